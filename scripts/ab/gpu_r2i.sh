cd $GRAFT_REPO_ROOT
python -c "import paper_2204_09131_b200.build as b; b.build()" > gpurun_out/r2i_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next3.py -x -q > gpurun_out/r2i_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2i_tests.log
timeout 300 python scripts/kernel_bench.py --target 2e11 > gpurun_out/r2i_kbench.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/r2i_kbench.jsonl'):
    d=json.loads(l); print(d['w'], round(d['kernel_ms'],3), round(d['frac_of_bruteforce_roofline'],3))
"
cat > /tmp/sweep_ab.py <<'PY'
import json, os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch, bench, paper_2204_09131_b200 as isy
r = bench.sweep_cfg3(isy, torch.cuda.current_stream(), 3)
print(json.dumps({"ms": r["ms_per_step"], "frac": r["roofline"]["frac"], "share": r["roofline"]["kernel_share_of_step"]}))
PY
timeout 300 python /tmp/sweep_ab.py 2>&1 | tail -1
for la in 8 16 32 64 128; do ISYCOS_LOOKAHEAD=$la timeout 120 python scripts/time_search.py cfg2 8 2>&1 | tail -1; done
for d in 2 4 8; do ISYCOS_BU_DEPTH=$d timeout 120 python scripts/time_search.py cfg2 8 2>&1 | tail -1; done
ISYCOS_PIPELINE=0 timeout 120 python scripts/time_search.py cfg2 8 2>&1 | tail -1
ISYCOS_LAT_WINDOWS=64 timeout 120 python scripts/time_search.py cfg2 8 2>&1 | tail -1
ISYCOS_LAT_SPLIT=0 timeout 120 python scripts/time_search.py cfg2 8 2>&1 | tail -1
