cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_search.py -m gpu -q -rf -x --timeout 600 -p no:cacheprovider > gpurun_out/gpu_search.log 2>&1; echo "search rc=$?"; tail -2 gpurun_out/gpu_search.log
for t in 16 32 64 128; do
  rm -f gpurun_out/trace_$t.txt
  ISYCOS_TREND_DEPTH=$t ISYCOS_TRACE=gpurun_out/trace_$t.txt timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_t$t.json 2>/dev/null
  echo "trend=$t $(python -c "import json;d=json.load(open('gpurun_out/bench_t$t.json'));print(d['ms_per_step'], d['e2e']['value'], d['host_ms_per_step'], d['rounds_per_step'], d['windows_per_s'])")"; grep "#" gpurun_out/trace_$t.txt | tail -1
done
