# warp-sorted kernel with G warps per window: parity (forced G = 1, 2, 4, auto) and the configs[3] 64-pair step
# A/B (auto vs G = 1), interleaved; launch list of 16 pairs with the auto G
cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r3d_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_wsgroup.py tests/test_gpu_parity.py -k "groups or warp_sorted" -q > $O/r3d_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/r3d_tests.log
for G in 0 1 0 1 0 1; do
  c4=$(ISYCOS_WS_GROUP=$G timeout 600 python scripts/measure_full.py cfg4 --pairs 64 --reps 3 2>&1 | python -c "
import json,sys
print([round(json.loads(l)['ms']) for l in sys.stdin if l.startswith('{')][1:])
")
  echo "ws_group $G cfg4 $c4"
done
for G in 0 1; do
  c2=$(ISYCOS_WS_GROUP=$G timeout 300 python scripts/time_search.py cfg2 6 2>&1 | tail -1 | cut -c1-60)
  echo "ws_group $G cfg2 $c2"
done
timeout 1200 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
  --log-file /tmp/r3d_launches.csv python scripts/measure_full.py cfg4 --pairs 16 > $O/r3d_ncu_launches.log 2>&1; echo "ncu launches rc=$?"
python scripts/ncu_summary.py launches /tmp/r3d_launches.csv $O/r3d_launches_cfg4_16pairs.md
