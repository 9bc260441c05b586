cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -x --timeout 900 -p no:cacheprovider > gpurun_out/gpu_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/gpu_parity.log
for mw in 33 65 257; do
  echo "wsorted_min_w=$mw"
  for w in 64 128 256; do ISYCOS_WSORTED_MIN_W=$mw timeout 300 python scripts/kernel_bench.py --target 1e11 --only $w 2>&1 | tail -1; done
  ISYCOS_WSORTED_MIN_W=$mw timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/bench_ws$mw.json 2>/dev/null
  echo "bench $(python -c "import json;d=json.load(open('gpurun_out/bench_ws$mw.json'));print(d['ms_per_step'], d['e2e']['value'], d['roofline']['paths'])")"
done
