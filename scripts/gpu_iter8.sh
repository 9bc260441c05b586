cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_search.py -m gpu -q -rf -x --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 300 python scripts/kernel_bench.py --target 1e11 > gpurun_out/kbench.jsonl 2>&1; echo "kbench rc=$?"; cat gpurun_out/kbench.jsonl
for f in 1 0; do
  ISYCOS_FUSED=$f timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_f$f.json 2>/dev/null
  echo "fused=$f $(python -c "import json;d=json.load(open('gpurun_out/bench_f$f.json'));print(d['ms_per_step'], d['e2e']['value'], d['host_ms_per_step'], d['rounds_per_step'], d['roofline']['paths'])")"
done
rm -f gpurun_out/trace.txt; ISYCOS_TRACE=gpurun_out/trace.txt timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; grep "#" gpurun_out/trace.txt | tail -1
