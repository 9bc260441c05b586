# One GPU-box pass (run via gpurun from the repo root): GPU parity tests, smoke, kernel microbench,
# bench (+ reference arm), the ncu launch list of the bench step and --set full captures of the kernels
# bench.py reports on.  Summaries: python scripts/ncu_summary.py {launches,rep,traffic} ...
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 1200 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 300 python scripts/kernel_bench.py --target 1e11 > gpurun_out/kbench.jsonl 2>&1; echo "kbench rc=$?"; cat gpurun_out/kbench.jsonl
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; cat gpurun_out/bench_ref.json
# ncu passes (each only after its command exited 0 without ncu, above)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ksg_tile|ksg_small|fused_sorted|warp_sorted" -s 300 -c 8 -o gpurun_out/prof_cfg2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc=$?"
timeout 300 python scripts/kernel_bench.py --only 4096 --reps 1 --target 1e11 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sorted_knn|sort_window" -s 2 -c 2 -o gpurun_out/prof_sweep4096 python scripts/kernel_bench.py --only 4096 --reps 1 --target 1e11 > gpurun_out/ncu3.log 2>&1; echo "ncu3 rc=$?"
