cd $GRAFT_REPO_ROOT
nproc > gpurun_out/r2a_nproc.txt; lscpu | head -20 >> gpurun_out/r2a_nproc.txt
timeout 600 python scripts/measure_full.py cfg4 --pairs 64 > gpurun_out/r2a_cfg4_64.jsonl 2>&1; echo "cfg4-64 rc=$?"
timeout 900 python scripts/measure_full.py cfg4 > gpurun_out/r2a_cfg4_full.jsonl 2>&1; echo "cfg4-full rc=$?"
timeout 600 python scripts/measure_full.py cfg5 --pairs 8 > gpurun_out/r2a_cfg5_8.jsonl 2>&1; echo "cfg5-8 rc=$?"
timeout 900 python scripts/measure_full.py cfg5 > gpurun_out/r2a_cfg5_full.jsonl 2>&1; echo "cfg5-full rc=$?"
tail -c 3000 gpurun_out/r2a_*.jsonl
