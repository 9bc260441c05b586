cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r2y_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_columns.py -q -x > $O/r2y_tests.log 2>&1; echo "column tests rc=$?"; tail -15 $O/r2y_tests.log
ISYCOS_COL_MIN_W=1024 timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x -k "sweep" > $O/r2y_fullsize.log 2>&1; echo "fullsize sweep (col 1024) rc=$?"; tail -2 $O/r2y_fullsize.log
cat > /tmp/sweep_ab.py <<'PY'
import json, os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch, bench, paper_2204_09131_b200 as isy
r = bench.sweep_cfg3(isy, torch.cuda.current_stream(), 3)
print(json.dumps({"ms": round(r["ms_per_step"], 2), "frac": round(r["roofline"]["frac"], 4)}))
PY
for C in 1073741824 1024 4096 16384 1073741824 1024 4096 16384; do
  echo "sweep col_min_w $C $(ISYCOS_COL_MIN_W=$C timeout 300 python /tmp/sweep_ab.py 2>&1 | tail -1)"
done
for C in 1073741824 1024; do
  for W in 1024 4096 16384; do
    ISYCOS_COL_MIN_W=$C timeout 300 python scripts/kernel_bench.py --only $W --reps 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kbench col $C w', d['w'], 'kernel_ms', round(d['kernel_ms'],3))"
  done
done
