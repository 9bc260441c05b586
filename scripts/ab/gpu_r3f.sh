# phase A two-sided scan with 16-byte pair loads (aligned blocks, self masked in the first block): parity of every
# sorted-path family, kernel bench, sweep, the ncu L1 breakdown of sorted_knn at w = 16,384, and the bench line
cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r3f_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next3.py tests/test_gpu_wsgroup.py tests/test_gpu_fullsize.py tests/test_gpu_t5.py -x -q > $O/r3f_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/r3f_tests.log
timeout 600 python scripts/kernel_bench.py > $O/r3f_kbench.jsonl 2>&1; echo "kbench rc=$?"
timeout 900 python bench.py > $O/r3f_bench.json 2> $O/r3f_bench.err; echo "bench rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:"sorted_knn" -c 1 -o /tmp/r3f_16384 \
  python scripts/kernel_bench.py --only 16384 --reps 1 --target 1e11 > $O/r3f_ncu_16384.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/r3f_16384.ncu-rep --page details --print-details all > $O/r3f_details_16384.txt 2>&1
