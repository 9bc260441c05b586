cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_search.py -m gpu -q -rf -x --timeout 600 -p no:cacheprovider > gpurun_out/gpu_search.log 2>&1; echo "search rc=$?"; tail -2 gpurun_out/gpu_search.log
rm -f gpurun_out/trace4.txt; ISYCOS_TRACE=gpurun_out/trace4.txt timeout 300 python bench.py --workload cfg4s --steps 2 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/bench_cfg4s.json 2>/dev/null
echo "cfg4s $(python -c "import json;d=json.load(open('gpurun_out/bench_cfg4s.json'));print(d['ms_per_step'], d['value'], d['windows_per_s'], d['host_ms_per_step'])")"; grep "#" gpurun_out/trace4.txt | tail -1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/bench_c2.json 2>/dev/null
echo "cfg2 $(python -c "import json;d=json.load(open('gpurun_out/bench_c2.json'));print(d['ms_per_step'], d['e2e']['value'])")"
