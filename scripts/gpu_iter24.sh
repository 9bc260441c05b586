cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_search.py -m gpu -q -rf -x --timeout 1200 -p no:cacheprovider -k "full_size" --durations=5 > gpurun_out/gpu_full.log 2>&1; echo "full rc=$?"; tail -12 gpurun_out/gpu_full.log
