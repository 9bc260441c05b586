cd $GRAFT_REPO_ROOT
python -c "import paper_2204_09131_b200.build as b; b.build()" > gpurun_out/r2b_build.log 2>&1
timeout 300 python __graft_entry__.py --smoke > gpurun_out/r2b_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q -k "not cfg4_full_size and not cfg5_prefix" > gpurun_out/r2b_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2b_gpu_tests.log
timeout 900 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/r2b_bench.err
