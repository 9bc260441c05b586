cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_search.py -m gpu -q -rf -x --timeout 900 -p no:cacheprovider -k "not cfg2_full and not cfg3 and not large_window" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
for lw in 0 100000; do ISYCOS_LAT_WINDOWS=$lw timeout 300 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/bench_lw$lw.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/bench_lw$lw.json'));print('lat_windows=$lw', round(d['ms_per_step'],1), 'host', round(d['host_ms_per_step'],1))"; done
rm -f gpurun_out/trace_cfg2.txt; ISYCOS_TRACE=gpurun_out/trace_cfg2.txt timeout 300 python bench.py --no-cpu-baseline --steps 1 --warmup 3 > /dev/null 2>&1
timeout 300 python scripts/kernel_bench.py --only 4096 --reps 1 > gpurun_out/plain_s4096.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"sorted_knn|sort_window" -s 2 -c 2 -o gpurun_out/prof_sorted4096 python scripts/kernel_bench.py --only 4096 --reps 1 > gpurun_out/ncu_sorted.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_sorted.log
