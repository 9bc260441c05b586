cd $GRAFT_REPO_ROOT
python -c "import paper_2204_09131_b200.build as b; b.build()" > gpurun_out/r2g_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_next3.py tests/test_gpu_search.py -x -q > gpurun_out/r2g_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2g_tests.log
for u in 1 0; do
  ISYCOS_SCAN_UNIFIED=$u timeout 300 python scripts/kernel_bench.py --target 2e11 > gpurun_out/r2g_kbench_u$u.jsonl 2>&1
done
cat > /tmp/sweep_ab.py <<'PY'
import json, os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch, bench, paper_2204_09131_b200 as isy
r = bench.sweep_cfg3(isy, torch.cuda.current_stream(), 3)
print(json.dumps({"ms": r["ms_per_step"], "frac": r["roofline"]["frac"], "share": r["roofline"]["kernel_share_of_step"]}))
PY
for u in 1 0; do for b in 1 0; do
  echo "unified=$u block=$b $(ISYCOS_SCAN_UNIFIED=$u ISYCOS_BLOCK_SORT=$b timeout 300 python /tmp/sweep_ab.py 2>&1 | tail -1)"
done; done | tee gpurun_out/r2g_sweep_ab.txt
ISYCOS_TRACE=gpurun_out/r2g_trace.txt timeout 300 python scripts/measure_full.py cfg4 --pairs 64 --reps 2 > gpurun_out/r2g_cfg4_64.jsonl 2>&1
ISYCOS_SCAN_UNIFIED=0 timeout 300 python scripts/measure_full.py cfg4 --pairs 64 --reps 2 > gpurun_out/r2g_cfg4_64_u0.jsonl 2>&1
for f in gpurun_out/r2g_cfg4*.jsonl; do python -c "
import json
for l in open('$f'):
    try:
        d=json.loads(l)
    except Exception:
        continue
    k=d['kernel']; print('$f', d['rep'], 'ms', round(d['ms']), 'host', round(k['host_ms']), 'rounds', k['rounds'])
"; done
grep -h "^#" gpurun_out/r2g_trace.txt
