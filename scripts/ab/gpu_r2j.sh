cd $GRAFT_REPO_ROOT
python -c "import paper_2204_09131_b200.build as b; b.build()" > gpurun_out/r2j_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_next3.py tests/test_gpu_fullsize.py -x -q -k "not cfg4_full" > gpurun_out/r2j_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r2j_tests.log
cat > /tmp/sweep_ab.py <<'PY'
import json, os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch, bench, paper_2204_09131_b200 as isy
r = bench.sweep_cfg3(isy, torch.cuda.current_stream(), 3)
print(json.dumps({"ms": r["ms_per_step"], "frac": r["roofline"]["frac"], "share": r["roofline"]["kernel_share_of_step"], "steps_per_point": r["roofline"]["scan_steps_per_point"]}))
PY
echo "inc on  $(timeout 300 python /tmp/sweep_ab.py 2>&1 | tail -1)"
echo "inc off $(ISYCOS_INCREMENTAL=0 timeout 300 python /tmp/sweep_ab.py 2>&1 | tail -1)"
echo "no block $(ISYCOS_BLOCK_SORT=0 timeout 300 python /tmp/sweep_ab.py 2>&1 | tail -1)"
timeout 300 python scripts/measure_full.py cfg4 --pairs 64 --reps 2 > gpurun_out/r2j_cfg4_64.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/r2j_cfg4_64.jsonl'):
    try:
        d=json.loads(l)
    except Exception:
        continue
    k=d['kernel']; print('cfg4', d['rep'], 'ms', round(d['ms']), 'host', round(k['host_ms']), 'inc', k['inc_windows'], k['eps_reused_points'])
"
