cd $GRAFT_REPO_ROOT
for i in 1 2 3; do timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/bench_b3.json 2>/dev/null
echo "bench $(python -c "import json;d=json.load(open('gpurun_out/bench_b3.json'));print(d['ms_per_step'], d['e2e']['value'], d['host_ms_per_step'], d['clocks'])")"; done
