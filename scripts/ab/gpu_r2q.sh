cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r2q_build.log 2>&1
rm -f /tmp/trd; ISYCOS_TRACE=/tmp/trd timeout 600 python scripts/measure_full.py cfg4 --pairs 64 --reps 3 > $O/r2q_cfg4.jsonl 2>&1
grep "^#" /tmp/trd > $O/r2q_trace_summary.txt
python -c "
import json
for l in open('$O/r2q_cfg4.jsonl'):
    try: d=json.loads(l)
    except Exception: continue
    print('cfg4 rep', d['rep'], 'ms', round(d['ms']), 'host', round(d['kernel']['host_ms']))
"
cat $O/r2q_trace_summary.txt
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_search.py tests/test_gpu_parity.py -q -x > $O/r2q_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/r2q_tests.log
