cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -x --timeout 900 -p no:cacheprovider > gpurun_out/gpu_seg.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/gpu_seg.log
timeout 300 python scripts/kernel_bench.py --target 1e11 > gpurun_out/kbench.jsonl 2>&1; echo "kbench rc=$?"; tail -4 gpurun_out/kbench.jsonl
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2>gpurun_out/bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['ms_per_step'], d['e2e']['value'], d['throughput_sweep']['ms_per_step'], d['throughput_sweep']['roofline']['frac'], d['multi_pair_search']['ms_per_step'])"
