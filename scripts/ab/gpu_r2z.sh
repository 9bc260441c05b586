cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r2z_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_columns.py -q -x > $O/r2z_tests.log 2>&1; echo "column tests rc=$?"; tail -3 $O/r2z_tests.log
cat > /tmp/sweep_ab.py <<'PY'
import json, os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch, bench, paper_2204_09131_b200 as isy
r = bench.sweep_cfg3(isy, torch.cuda.current_stream(), 3)
print(json.dumps({"ms": round(r["ms_per_step"], 2), "frac": round(r["roofline"]["frac"], 4)}))
PY
for C in 1073741824 16384 4096 1073741824 16384 4096; do
  echo "sweep col_min_w $C $(ISYCOS_COL_MIN_W=$C timeout 300 python /tmp/sweep_ab.py 2>&1 | tail -1)"
done
for C in 1073741824 1024; do
  for W in 4096 16384; do
    ISYCOS_COL_MIN_W=$C timeout 300 python scripts/kernel_bench.py --only $W --reps 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kbench col $C w', d['w'], 'kernel_ms', round(d['kernel_ms'],3))"
  done
done
ISYCOS_COL_MIN_W=1024 timeout 900 ncu --set full --clock-control none -k regex:"sorted_knn" -c 1 -o /tmp/r2z_col python scripts/kernel_bench.py --only 16384 --reps 1 --target 2e10 > /dev/null 2>&1
python scripts/ncu_summary.py rep /tmp/r2z_col.ncu-rep $O/r2z_ncu_col16384.md
python scripts/ncu_summary.py opcodes /tmp/r2z_col.ncu-rep sorted_knn $O/r2z_col_opcodes.txt
grep -E "Duration|Issue Slots|Active Threads|Achieved Occ|No Eligible|Warp Cycles" $O/r2z_ncu_col16384.md; head -12 $O/r2z_col_opcodes.txt
