cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r3a_build.log 2>&1
# host pool: yields a worker spins before sleeping (wake-up latency vs. CPU burn)
for SP in 20000 200000 2000000 20000 200000 2000000; do
  rm -f /tmp/trd
  c4=$(ISYCOS_POOL_SPIN=$SP ISYCOS_TRACE=/tmp/trd timeout 600 python scripts/measure_full.py cfg4 --pairs 64 --reps 3 2>&1 | python -c "
import json,sys
print([round(json.loads(l)['ms']) for l in sys.stdin if l.startswith('{')][1:])
")
  echo "spin $SP cfg4 $c4 $(grep '^# host' /tmp/trd | tail -1 | cut -c1-150)"
  c2=$(ISYCOS_POOL_SPIN=$SP timeout 300 python scripts/time_cfg2.py --reps 5 2>&1 | python -c "
import json,sys
print([round(json.loads(l)['ms'],1) for l in sys.stdin if l.startswith('{')][1:])
")
  echo "spin $SP cfg2 $c2"
done
