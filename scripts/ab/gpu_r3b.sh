cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r3b_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_next3.py tests/test_gpu_t5.py tests/test_gpu_search.py -q -x > $O/r3b_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/r3b_tests.log
# latency kernel: 4 lanes per point up to w = 128 (default) vs 8 lanes everywhere
for L4 in 128 0 128 0; do
  c4=$(ISYCOS_LAT_LANES4_MAX_W=$L4 timeout 600 python scripts/measure_full.py cfg4 --pairs 64 --reps 3 2>&1 | python -c "
import json,sys
print([round(json.loads(l)['ms']) for l in sys.stdin if l.startswith('{')][1:])
")
  c2=$(ISYCOS_LAT_LANES4_MAX_W=$L4 timeout 300 python scripts/time_cfg2.py --reps 5 2>&1 | python -c "
import json,sys
print([round(json.loads(l)['ms'],1) for l in sys.stdin if l.startswith('{')][1:])
")
  echo "lanes4_max_w $L4 cfg4 $c4 cfg2 $c2"
done
for L4 in 128 0; do
  ISYCOS_LAT_LANES4_MAX_W=$L4 timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file /tmp/r3b_l$L4.csv python scripts/measure_full.py cfg4 --pairs 16 > /dev/null 2>&1
  python scripts/ncu_summary.py launches /tmp/r3b_l$L4.csv $O/r3b_launches_lanes4_$L4.md
  echo "lanes4_max_w $L4: $(grep ksg_lat $O/r3b_launches_lanes4_$L4.md)"
done
# host pool spin (yields before a worker sleeps): 20000 default; 200000 / 2000000 measured worse (r3a)
for SP in 2000 200 20000 2000 200; do
  c4=$(ISYCOS_POOL_SPIN=$SP timeout 600 python scripts/measure_full.py cfg4 --pairs 64 --reps 3 2>&1 | python -c "
import json,sys
print([round(json.loads(l)['ms']) for l in sys.stdin if l.startswith('{')][1:])
")
  echo "spin $SP cfg4 $c4"
done
