cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -x --timeout 600 -p no:cacheprovider > gpurun_out/gpu_parity.log 2>&1; echo "parity rc=$?"; tail -8 gpurun_out/gpu_parity.log
timeout 300 python scripts/kernel_bench.py --target 1e11 > gpurun_out/kbench.jsonl 2>&1; echo "kbench rc=$?"; cat gpurun_out/kbench.jsonl
ISYCOS_FUSED=0 timeout 300 python scripts/kernel_bench.py --target 1e11 > gpurun_out/kbench_nofused.jsonl 2>&1; echo "kbench nofused rc=$?"; cat gpurun_out/kbench_nofused.jsonl
for cfg in "4 64" "4 32" "4 16" "3 32" "2 64"; do set -- $cfg
  ISYCOS_BU_DEPTH=$1 ISYCOS_LOOKAHEAD=$2 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_d$1_l$2.json 2>/dev/null
  echo "D=$1 LA=$2 $(python -c "import json;d=json.load(open('gpurun_out/bench_d$1_l$2.json'));print(d['ms_per_step'], d['e2e']['value'], d['host_ms_per_step'], d['rounds_per_step'], d['roofline']['paths'])")"
done
