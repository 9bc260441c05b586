cd $GRAFT_REPO_ROOT
nproc; lscpu | grep "Model name"
timeout 900 python -m pytest tests/test_gpu_search.py -m gpu -q -rf -x --timeout 600 -p no:cacheprovider -k "cfg4 or multi or cfg5" > gpurun_out/gpu_search.log 2>&1; echo "search rc=$?"; tail -2 gpurun_out/gpu_search.log
for t in 0 1; do
ISYCOS_HOST_THREADS=$t timeout 900 python bench.py --workload cfg4s --steps 1 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/bench_cfg4s_t$t.json 2>/dev/null
echo "threads=$t $(python -c "import json;d=json.load(open('gpurun_out/bench_cfg4s_t$t.json'));print(d['ms_per_step'], d['value'], d['windows_per_s'], d['host_ms_per_step'], d['rounds_per_step'])")"
done
