cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -x --timeout 300 -p no:cacheprovider -k "cfg1 or debug or device" > gpurun_out/gpu_sub.log 2>&1; echo "sub rc=$?"; tail -2 gpurun_out/gpu_sub.log
timeout 600 python bench.py > gpurun_out/bench.json 2>gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -2 gpurun_out/bench.err
