cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -x --timeout 900 -p no:cacheprovider > gpurun_out/gpu_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/gpu_parity.log
for sm in 0 1; do
  ISYCOS_SCAN_MODE=$sm timeout 300 python scripts/kernel_bench.py --target 1e11 --only 1024 > gpurun_out/kb_sm$sm.jsonl 2>&1
  ISYCOS_SCAN_MODE=$sm timeout 300 python scripts/kernel_bench.py --target 1e11 --only 4096 >> gpurun_out/kb_sm$sm.jsonl 2>&1
  ISYCOS_SCAN_MODE=$sm timeout 300 python scripts/kernel_bench.py --target 1e11 --only 16384 >> gpurun_out/kb_sm$sm.jsonl 2>&1
  echo "scan_mode=$sm"; cat gpurun_out/kb_sm$sm.jsonl
  ISYCOS_SCAN_MODE=$sm timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_sm$sm.json 2>gpurun_out/bench_sm$sm.err
  echo "bench scan_mode=$sm $(python -c "import json;d=json.load(open('gpurun_out/bench_sm$sm.json'));print(d['ms_per_step'], d['e2e']['value'], d['throughput_sweep'])")"
done
