cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -x --timeout 900 -p no:cacheprovider -k "maximum" > gpurun_out/gpu_max.log 2>&1; echo "max rc=$?"; tail -2 gpurun_out/gpu_max.log
timeout 900 python bench.py --workload cfg4s --steps 1 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/bench_cfg4s.json 2>gpurun_out/bench_cfg4s.err; echo "cfg4s rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_cfg4s.json'));print(d['ms_per_step'], d['value'], d['windows_per_s'], d['host_ms_per_step'], d['rounds_per_step'], d['roofline']['path'], d['roofline']['frac'], d['roofline']['paths'])"
