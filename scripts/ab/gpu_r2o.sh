cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r2o_build.log 2>&1
rm -f /tmp/trd; ISYCOS_TRACE=/tmp/trd timeout 600 python scripts/measure_full.py cfg4 --pairs 64 --reps 2 > $O/r2o_cfg4.jsonl 2>&1
grep "^#" /tmp/trd > $O/r2o_trace_summary.txt
awk '!/^#/ {c=($4>100000)?"big":(($4>2000)?"mid":"small"); n[c]++; h[c]+=$2; s[c]+=$3; a[c]+=$7; m[c]+=$8; w[c]+=$4} END {for (k in n) print k, n[k], "rounds; windows", w[k], "host-since-submit ms", h[k], "submit ms", s[k], "advance ms", a[k], "assemble ms", m[k]}' /tmp/trd >> $O/r2o_trace_summary.txt
python -c "
import json
for l in open('$O/r2o_cfg4.jsonl'):
    try: d=json.loads(l)
    except Exception: continue
    print('cfg4 rep', d['rep'], 'ms', round(d['ms']), 'host', round(d['kernel']['host_ms']))
"
cat $O/r2o_trace_summary.txt
timeout 1500 python -m pytest tests -m gpu -q -x > $O/r2o_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 $O/r2o_gpu_tests.log
