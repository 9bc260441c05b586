cd $GRAFT_REPO_ROOT
for w in 512 1024 4096 16384; do timeout 300 python scripts/kernel_bench.py --target 1e11 --only $w 2>&1 | tail -1 | cut -c1-110; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_search.py -m gpu -q -rf -x --timeout 900 -p no:cacheprovider > gpurun_out/gpu_mg.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/gpu_mg.log
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -1
