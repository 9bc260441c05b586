cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_search.py -m gpu -q -rf -x --timeout 900 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/bench_lat.json 2>/dev/null
echo "bench $(python -c "import json;d=json.load(open('gpurun_out/bench_lat.json'));print(d['ms_per_step'], d['e2e']['value'], d['host_ms_per_step'], d['roofline']['paths'])")"
for cfg in "3 32" "2 32" "4 16"; do set -- $cfg
  ISYCOS_BU_DEPTH=$1 ISYCOS_LOOKAHEAD=$2 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/bench_d$1_l$2.json 2>/dev/null
  echo "D=$1 LA=$2 $(python -c "import json;d=json.load(open('gpurun_out/bench_d$1_l$2.json'));print(d['ms_per_step'], d['e2e']['value'], d['host_ms_per_step'], d['rounds_per_step'])")"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
