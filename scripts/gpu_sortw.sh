cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -x --timeout 600 -p no:cacheprovider -k "size_classes or tie or ksg2 or cfg1 or segments or cfg3 or warp_sorted" > gpurun_out/gpu_s.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/gpu_s.log
timeout 300 python scripts/kernel_bench.py --target 1e11 > gpurun_out/kbench.jsonl 2>&1; echo "kbench rc=$?"; cat gpurun_out/kbench.jsonl
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2>gpurun_out/bench.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print(d['ms_per_step'], d['e2e']['value'], d['throughput_sweep']['ms_per_step'], d['throughput_sweep']['roofline']['frac'], d['multi_pair_search']['ms_per_step'])"
