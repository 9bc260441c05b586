cd $GRAFT_REPO_ROOT
python -c "import paper_2204_09131_b200.build as b; b.build()" > gpurun_out/r2c_build.log 2>&1
ISYCOS_TRACE=gpurun_out/r2c_trace.txt timeout 300 python scripts/measure_full.py cfg4 --pairs 64 --reps 2 > gpurun_out/r2c_cfg4_64.jsonl 2>&1; echo "trace rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/r2c_launches.csv python scripts/measure_full.py cfg4 --pairs 16 > gpurun_out/r2c_ncu1.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"warp_sorted|sorted_knn|sort_window|fused_sorted|ksg_tile|ksg_small" -s 3000 -c 12 -o gpurun_out/r2c_prof_cfg4 python scripts/measure_full.py cfg4 --pairs 16 > gpurun_out/r2c_ncu2.log 2>&1; echo "ncu2 rc=$?"
ls -la gpurun_out/
