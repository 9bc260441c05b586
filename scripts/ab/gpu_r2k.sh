cd $GRAFT_REPO_ROOT
python -c "import paper_2204_09131_b200.build as b; b.build()" > gpurun_out/r2k_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_next3.py tests/test_gpu_fullsize.py -x -q -k "not cfg4_full" > gpurun_out/r2k_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2k_tests.log
cat > /tmp/sweep_ab.py <<'PY'
import json, os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch, bench, paper_2204_09131_b200 as isy
r = bench.sweep_cfg3(isy, torch.cuda.current_stream(), 3)
print(json.dumps({"ms": r["ms_per_step"], "frac": r["roofline"]["frac"], "steps_per_point": r["roofline"]["scan_steps_per_point"]}))
PY
for c in 2 4 8 16; do echo "chain $c $(ISYCOS_INC_CHAIN=$c timeout 300 python /tmp/sweep_ab.py 2>&1 | tail -1)"; done
echo "inc off $(ISYCOS_INCREMENTAL=0 timeout 300 python /tmp/sweep_ab.py 2>&1 | tail -1)"
