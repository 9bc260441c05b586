cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_search.py -m gpu -q -rf -x --timeout 600 -p no:cacheprovider -k "size_classes or cfg1 or cfg2_full or tie" > gpurun_out/gpu_zc.log 2>&1; echo "parity(zc default) rc=$?"; tail -2 gpurun_out/gpu_zc.log
ISYCOS_ZC_DESC=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_search.py -m gpu -q -rf -x --timeout 600 -p no:cacheprovider -k "size_classes or cfg1 or cfg2_full or tie" > gpurun_out/gpu_zc1.log 2>&1; echo "parity(zc=1) rc=$?"; tail -2 gpurun_out/gpu_zc1.log
for z in 0 1 0 1; do
  ISYCOS_ZC_DESC=$z timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/bench_zc.json 2>/dev/null
  echo "zc=$z $(python -c "import json;d=json.load(open('gpurun_out/bench_zc.json'));print(d['ms_per_step'], d['e2e']['value'], d['host_ms_per_step'])")"
done
