cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_search.py -m gpu -q -rf -x --timeout 600 -p no:cacheprovider -k "cfg1 or debug or size_classes or tie or ksg2 or cfg2_full" > gpurun_out/gpu_sub.log 2>&1; echo "sub rc=$?"; tail -3 gpurun_out/gpu_sub.log
rm -f gpurun_out/trace.txt; ISYCOS_TRACE=gpurun_out/trace.txt timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_trace.json 2>&1; echo "trace rc=$?"; grep "#" gpurun_out/trace.txt | tail -2
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
bash scripts/gpu_sweep_minw.sh
