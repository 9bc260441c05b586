# speculation parameter sweep on the cfg2 bench + a per-round trace
cd $GRAFT_REPO_ROOT
for d in 1 2 3 4; do
  for la in 64 256; do
    ISYCOS_BU_DEPTH=$d ISYCOS_LOOKAHEAD=$la timeout 300 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/sweep_d${d}_la${la}.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/sweep_d${d}_la${la}.json'));print('depth=$d la=$la', round(d['ms_per_step'],1), 'rounds', d['rounds_per_step'], 'host', round(d['host_ms_per_step'],1), 'kshare', round(d['roofline']['kernel_share_of_step'],3), 'evalTc', round(d['roofline']['evaluated_compares_per_step']/1e12,4))"
  done
done
ISYCOS_TRACE=gpurun_out/trace_cfg2.txt timeout 300 python bench.py --no-cpu-baseline --steps 1 --warmup 3 > /dev/null 2>&1
wc -l gpurun_out/trace_cfg2.txt
timeout 300 python scripts/kernel_bench.py --target 1e11 > gpurun_out/kbench.jsonl 2>&1; cat gpurun_out/kbench.jsonl
