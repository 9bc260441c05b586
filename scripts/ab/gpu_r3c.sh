cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r3c_build.log 2>&1
# host pool size with the asynchronous submit thread (16 cores): leave a core for the submit thread?
for HT in 16 15 14 12 16 15 14 12; do
  rm -f /tmp/trd
  c4=$(ISYCOS_HOST_THREADS=$HT ISYCOS_TRACE=/tmp/trd timeout 600 python scripts/measure_full.py cfg4 --pairs 64 --reps 3 2>&1 | python -c "
import json,sys
print([round(json.loads(l)['ms']) for l in sys.stdin if l.startswith('{')][1:])
")
  echo "threads $HT cfg4 $c4 $(grep '^# host' /tmp/trd | tail -1 | cut -c1-150)"
done
for BT in 16 8 4 16 8 4; do
  c4=$(ISYCOS_BIN_THREADS=$BT timeout 600 python scripts/measure_full.py cfg4 --pairs 64 --reps 3 2>&1 | python -c "
import json,sys
print([round(json.loads(l)['ms']) for l in sys.stdin if l.startswith('{')][1:])
")
  echo "bin_threads $BT cfg4 $c4"
done
