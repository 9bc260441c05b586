# pair loads gated to global P2 with w >= 2,048 (shared-memory scans keep 8-byte loads): parity, kernel bench, bench
# sorted-path family, kernel bench, sweep, the ncu L1 breakdown of sorted_knn at w = 16,384, and the bench line
cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r3g_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next3.py tests/test_gpu_wsgroup.py tests/test_gpu_fullsize.py tests/test_gpu_t5.py tests/test_gpu_ballot.py -x -q > $O/r3g_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/r3g_tests.log
timeout 600 python scripts/kernel_bench.py > $O/r3g_kbench.jsonl 2>&1; echo "kbench rc=$?"
timeout 900 python bench.py > $O/r3g_bench.json 2> $O/r3g_bench.err; echo "bench rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:"sorted_knn" -c 1 -o /tmp/r3g_16384 \
  python scripts/kernel_bench.py --only 16384 --reps 1 --target 1e11 > $O/r3g_ncu_16384.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/r3g_16384.ncu-rep --page details --print-details all > $O/r3g_details_16384.txt 2>&1
