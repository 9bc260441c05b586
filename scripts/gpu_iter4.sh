cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rf -x --timeout 900 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 300 python scripts/kernel_bench.py --target 1e11 > gpurun_out/kbench.jsonl 2>&1; echo "kbench rc=$?"; cat gpurun_out/kbench.jsonl
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 300 python scripts/kernel_bench.py --only 4096 --reps 1 --target 1e11 > gpurun_out/plain_s4096.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"sorted_knn|sort_window" -s 2 -c 2 -o gpurun_out/prof_sorted4096d python scripts/kernel_bench.py --only 4096 --reps 1 --target 1e11 > gpurun_out/ncu_sorted.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_sorted.log
