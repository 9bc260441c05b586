cd $GRAFT_REPO_ROOT
for mw in 1073741824 129 65 33; do
  ISYCOS_FUSED_SMALL_MIN_W=$mw timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/bench_fs$mw.json 2>/dev/null
  echo "fused_small_min_w=$mw $(python -c "import json;d=json.load(open('gpurun_out/bench_fs$mw.json'));print(d['ms_per_step'], d['e2e']['value'], d['roofline']['path'], d['roofline']['frac'])")"
done
ISYCOS_FUSED_SMALL_MIN_W=65 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_search.py -m gpu -q -rf -x --timeout 600 -p no:cacheprovider -k "size_classes or tie or cfg1 or cfg2_full" > gpurun_out/gpu_fs.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/gpu_fs.log
