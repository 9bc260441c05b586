cd $GRAFT_REPO_ROOT
python -c "import paper_2204_09131_b200.build as b; b.build()" > gpurun_out/r2d_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_next3.py tests/test_gpu_parity.py tests/test_gpu_search.py -x -q > gpurun_out/r2d_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2d_tests.log
ISYCOS_TRACE=gpurun_out/r2d_trace.txt timeout 300 python scripts/measure_full.py cfg4 --pairs 64 --reps 2 > gpurun_out/r2d_cfg4_64.jsonl 2>&1; echo "trace rc=$?"
ISYCOS_BLOCK_SORT=0 timeout 300 python scripts/measure_full.py cfg4 --pairs 64 --reps 2 > gpurun_out/r2d_cfg4_64_noblock.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file /tmp/r2d_launches.csv python scripts/measure_full.py cfg4 --pairs 16 > gpurun_out/r2d_ncu1.log 2>&1; echo "ncu1 rc=$?"
python scripts/ncu_summary.py launches /tmp/r2d_launches.csv gpurun_out/r2d_launches_cfg4.md; gzip -c /tmp/r2d_launches.csv > gpurun_out/r2d_launches.csv.gz
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"warp_sorted|sorted_knn|sort_window|fused_sorted|ksg_tile|ksg_small" -s 3000 -c 6 -o /tmp/r2d_prof_cfg4 python scripts/measure_full.py cfg4 --pairs 16 > gpurun_out/r2d_ncu2.log 2>&1; echo "ncu2 rc=$?"
python scripts/ncu_summary.py rep /tmp/r2d_prof_cfg4.ncu-rep gpurun_out/r2d_ncu_cfg4.md
python scripts/ncu_summary.py issue /tmp/r2d_prof_cfg4.ncu-rep cfg4_mix ".*" gpurun_out/r2d_issue.json
ls -la gpurun_out/; du -sh gpurun_out
