cd $GRAFT_REPO_ROOT
python -c "import paper_2204_09131_b200.build as b; b.build()" > gpurun_out/r2h_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next3.py tests/test_gpu_search.py -x -q > gpurun_out/r2h_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2h_tests.log
timeout 300 python scripts/kernel_bench.py --target 2e11 > gpurun_out/r2h_kbench.jsonl 2>&1
cat > /tmp/sweep_ab.py <<'PY'
import json, os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch, bench, paper_2204_09131_b200 as isy
r = bench.sweep_cfg3(isy, torch.cuda.current_stream(), 3)
print(json.dumps({"ms": r["ms_per_step"], "frac": r["roofline"]["frac"], "share": r["roofline"]["kernel_share_of_step"]}))
PY
timeout 300 python /tmp/sweep_ab.py 2>&1 | tail -1 | tee gpurun_out/r2h_sweep.txt
timeout 300 python scripts/measure_full.py cfg4 --pairs 64 --reps 2 > gpurun_out/r2h_cfg4_64.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/r2h_cfg4_64.jsonl'):
    try:
        d=json.loads(l)
    except Exception:
        continue
    k=d['kernel']; print('cfg4', d['rep'], 'ms', round(d['ms']), 'host', round(k['host_ms']), 'rounds', k['rounds'])
"
python -c "
import json
for l in open('gpurun_out/r2h_kbench.jsonl'):
    d=json.loads(l); print(d['w'], round(d['kernel_ms'],3), round(d['frac_of_bruteforce_roofline'],3))
"
