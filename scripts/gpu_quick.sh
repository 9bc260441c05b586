# parity of the sorted paths + kernel microbench + bench (a quick pass after a kernel change)
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -x --timeout 900 -p no:cacheprovider > gpurun_out/gpu_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/gpu_parity.log
timeout 300 python scripts/kernel_bench.py --target 1e11 > gpurun_out/kbench.jsonl 2>&1; echo "kbench rc=$?"; cat gpurun_out/kbench.jsonl
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2>gpurun_out/bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['throughput_sweep']['ms_per_step'], d['throughput_sweep']['roofline'])"
