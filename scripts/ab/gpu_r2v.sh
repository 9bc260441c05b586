cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r2v_build.log 2>&1
# configs[1] single-pair search: BU climbs on the host pool (default) vs serial
for PC in 1 0 1 0; do
  ISYCOS_PAR_CLIMBS=$PC timeout 300 python scripts/time_cfg2.py --reps 6 2>&1 | python -c "
import json,sys
r=[json.loads(l) for l in sys.stdin if l.startswith('{')]
print('par_climbs $PC cfg2 ms', [round(d['ms'],1) for d in r[1:]], 'host', [round(d['host_ms'],1) for d in r[1:]], 'results', r[-1]['results'])
"
done
rm -f /tmp/tr2; ISYCOS_TRACE=/tmp/tr2 timeout 300 python scripts/time_cfg2.py --reps 3 > /dev/null 2>&1; grep "^#" /tmp/tr2 | tail -2
timeout 1500 python -m pytest tests/test_gpu_search.py tests/test_gpu_t5.py -q -x > $O/r2v_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/r2v_tests.log
timeout 600 python scripts/measure_full.py cfg4 --pairs 64 --reps 3 2>&1 | python -c "
import json,sys
print('cfg4', [round(json.loads(l)['ms']) for l in sys.stdin if l.startswith('{')])
"
