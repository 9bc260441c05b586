cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r2w_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_next3.py tests/test_gpu_parity.py tests/test_gpu_t5.py tests/test_gpu_ballot.py -q -x > $O/r2w_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/r2w_tests.log
# tiny latency-mode windows (w <= 32) warp-per-window inside the latency launch (default) vs 8 lanes per point
for T in 32 0 32 0; do
  c4=$(ISYCOS_LAT_TINY_MAX_W=$T timeout 600 python scripts/measure_full.py cfg4 --pairs 64 --reps 3 2>&1 | python -c "
import json,sys
ms=[json.loads(l)['ms'] for l in sys.stdin if l.startswith('{')]
print([round(m) for m in ms[1:]])
")
  c2=$(ISYCOS_LAT_TINY_MAX_W=$T timeout 300 python scripts/time_cfg2.py --reps 6 2>&1 | python -c "
import json,sys
ms=[json.loads(l)['ms'] for l in sys.stdin if l.startswith('{')]
print([round(m,1) for m in ms[1:]])
")
  echo "tiny_max_w $T cfg4 $c4 cfg2 $c2"
done
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file /tmp/r2w_cfg2_launches.csv python scripts/time_cfg2.py --reps 1 > /dev/null 2>&1
python scripts/ncu_summary.py launches /tmp/r2w_cfg2_launches.csv $O/r2w_launches_cfg2.md; head -12 $O/r2w_launches_cfg2.md
