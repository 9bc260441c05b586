# one iteration: parity tests (FULL=1 for all), kernel bench, bench (+trace)
cd $GRAFT_REPO_ROOT
if [ "${FULL:-0}" = "1" ]; then SEL=""; else SEL="not cfg2_full and not cfg3"; fi
timeout 1500 python -m pytest tests -m gpu -q -rf -x --timeout 900 -p no:cacheprovider -k "$SEL" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/gpu_tests.log
timeout 300 python scripts/kernel_bench.py --target 1e11 > gpurun_out/kbench.jsonl 2>&1; echo "kbench rc=$?"; cat gpurun_out/kbench.jsonl
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
rm -f gpurun_out/trace_cfg2.txt; ISYCOS_TRACE=gpurun_out/trace_cfg2.txt timeout 300 python bench.py --no-cpu-baseline --steps 1 --warmup 3 > /dev/null 2>&1
