cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_search.py -m gpu -q -rf -x --timeout 600 -p no:cacheprovider -k "cfg1_search or cfg2" > gpurun_out/gpu_search.log 2>&1; echo "search rc=$?"; tail -2 gpurun_out/gpu_search.log
for rr in 1000000 8 2; do
  ISYCOS_RING_RANK=$rr timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/bench_rr$rr.json 2>/dev/null
  echo "ring_rank=$rr $(python -c "import json;d=json.load(open('gpurun_out/bench_rr$rr.json'));print(d['ms_per_step'], d['e2e']['value'], d['host_ms_per_step'], d['rounds_per_step'])")"
done
