cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -x --timeout 600 -p no:cacheprovider -k "warp_sorted or size_classes or cfg1" > gpurun_out/gpu_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/gpu_parity.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/bench_lat.json 2>/dev/null
echo "bench $(python -c "import json;d=json.load(open('gpurun_out/bench_lat.json'));print(d['ms_per_step'], d['e2e']['value'], d['roofline']['paths'])")"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fused_sorted|warp_sorted|ksg_tile|ksg_small" -s 300 -c 8 -o gpurun_out/prof_cfg2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc=$?"
timeout 300 python scripts/kernel_bench.py --target 1e11 --only 4096 --reps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sorted_knn|sort_window" -s 2 -c 2 -o gpurun_out/prof_sweep4096 python scripts/kernel_bench.py --only 4096 --reps 1 --target 1e11 > gpurun_out/ncu3.log 2>&1; echo "ncu3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"warp_sorted" -s 1 -c 1 -o gpurun_out/prof_ws256 python scripts/kernel_bench.py --only 256 --reps 1 --target 1e11 > gpurun_out/ncu4.log 2>&1; echo "ncu4 rc=$?"
