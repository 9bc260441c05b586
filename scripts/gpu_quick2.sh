cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_search.py -m gpu -q -rf -x --timeout 600 -p no:cacheprovider -k "size_classes or tie or ksg2 or cfg1 or cfg2_full or segments" > gpurun_out/gpu_q.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/gpu_q.log
for i in 1 2 3; do timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/bench_q.json 2>/dev/null
echo "bench $(python -c "import json;d=json.load(open('gpurun_out/bench_q.json'));print(d['ms_per_step'], d['e2e']['value'], d['roofline']['paths']['sorted_marginal']['kernel_ms'])")"; done
