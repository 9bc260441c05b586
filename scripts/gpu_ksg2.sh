cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_search.py -m gpu -q -rf --timeout 600 -p no:cacheprovider -k "ksg2 or brute" > gpurun_out/gpu_ksg2.log 2>&1; echo "ksg2 rc=$?"; tail -15 gpurun_out/gpu_ksg2.log
timeout 1200 python -m pytest tests -m gpu -q -rf --timeout 900 -p no:cacheprovider -k "not ksg2 and not brute" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
rm -f gpurun_out/trace.txt; ISYCOS_TRACE=gpurun_out/trace.txt timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_trace.json 2>&1; echo "trace rc=$?"; tail -3 gpurun_out/trace.txt
