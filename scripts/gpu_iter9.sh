cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_search.py -m gpu -q -rf -x --timeout 600 -p no:cacheprovider > gpurun_out/gpu_search.log 2>&1; echo "search rc=$?"; tail -3 gpurun_out/gpu_search.log
for pl in 1 0; do
  ISYCOS_PIPELINE=$pl timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_p$pl.json 2>/dev/null
  echo "pipeline=$pl $(python -c "import json;d=json.load(open('gpurun_out/bench_p$pl.json'));print(d['ms_per_step'], d['e2e']['value'], d['host_ms_per_step'], d['rounds_per_step'])")"
done
for la in 16 64; do
  ISYCOS_LOOKAHEAD=$la timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_la$la.json 2>/dev/null
  echo "la=$la $(python -c "import json;d=json.load(open('gpurun_out/bench_la$la.json'));print(d['ms_per_step'], d['e2e']['value'], d['host_ms_per_step'], d['rounds_per_step'])")"
done
rm -f gpurun_out/trace.txt; ISYCOS_TRACE=gpurun_out/trace.txt timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; grep "#" gpurun_out/trace.txt | tail -1
