cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r2p_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ballot.py -q > $O/r2p_ballot_tests.log 2>&1; echo "ballot tests rc=$?"; tail -2 $O/r2p_ballot_tests.log
# a4 count forms on the warp-per-window brute kernel: per-lane predicated adds (mode 1) vs warp ballot (mode 3)
for M in 1 3 1 3; do
  for W in 32 64; do
    ISYCOS_KNN_MODE=$M timeout 300 python scripts/kernel_bench.py --only $W --reps 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kbench mode $M w', d['w'], 'kernel_ms', round(d['kernel_ms'],3))"
  done
done | tee $O/r2p_ballot_kbench.txt
for M in 1 3; do
  ISYCOS_KNN_MODE=$M timeout 600 ncu --set full --clock-control none -k regex:ksg_small -c 1 -o /tmp/r2p_small_m$M python scripts/kernel_bench.py --only 64 --reps 1 --target 1e10 > $O/r2p_ncu_m$M.log 2>&1
  python scripts/ncu_summary.py rep /tmp/r2p_small_m$M.ncu-rep $O/r2p_ncu_small_mode$M.md
done
