cd $GRAFT_REPO_ROOT
python scripts/kernel_bench.py > gpurun_out/kbench.jsonl 2> gpurun_out/kbench.err; echo "kbench rc=$?"; cat gpurun_out/kbench.jsonl
python bench.py --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "bench rc=$?"; cat gpurun_out/bench2.json
python scripts/kernel_bench.py --only 4096 --reps 1 > gpurun_out/plain4096.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:ksg_tile_kernel -s 1 -c 1 -o gpurun_out/prof_tile4096 python scripts/kernel_bench.py --only 4096 --reps 1 > gpurun_out/ncu_t.log 2>&1; echo "ncu tile rc=$?"
python scripts/kernel_bench.py --only 128 --reps 1 > gpurun_out/plain128.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:ksg_small_kernel -s 1 -c 1 -o gpurun_out/prof_small128 python scripts/kernel_bench.py --only 128 --reps 1 > gpurun_out/ncu_s.log 2>&1; echo "ncu small rc=$?"
