cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r2r_build.log 2>&1
rm -f /tmp/tr2; ISYCOS_TRACE=/tmp/tr2 timeout 300 python scripts/time_cfg2.py --reps 5 > $O/r2r_cfg2.jsonl 2>&1
cat $O/r2r_cfg2.jsonl
grep "^#" /tmp/tr2 | tail -2
awk '!/^#/ {c=($4>256)?"gt256":(($4>32)?"33-256":"le32"); n[c]++; h[c]+=$2; s[c]+=$3; a[c]+=$7; w[c]+=$4} END {for (k in n) print k, n[k], "rounds; windows", w[k], "host-since-submit ms", h[k], "submit ms", s[k], "advance ms", a[k]}' /tmp/tr2
cp /tmp/tr2 $O/r2r_cfg2_trace.txt
timeout 900 nsys --version > /dev/null 2>&1 || true
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file /tmp/r2r_cfg2_launches.csv python scripts/time_cfg2.py --reps 1 > $O/r2r_ncu.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py launches /tmp/r2r_cfg2_launches.csv $O/r2r_launches_cfg2.md
head -30 $O/r2r_launches_cfg2.md
rm -f /tmp/trd; ISYCOS_TRACE=/tmp/trd timeout 600 python scripts/measure_full.py cfg4 --pairs 64 --reps 3 > $O/r2r_cfg4.jsonl 2>&1
python -c "
import json
for l in open('$O/r2r_cfg4.jsonl'):
    try: d=json.loads(l)
    except Exception: continue
    print('cfg4 rep', d['rep'], 'ms', round(d['ms']), 'host', round(d['kernel']['host_ms']))
"
grep "^#" /tmp/trd | tail -2
