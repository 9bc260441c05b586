cd $GRAFT_REPO_ROOT
for am in 0 256 100000; do
  ISYCOS_AUX_MIN_WINDOWS=$am timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/bench_am$am.json 2>/dev/null
  echo "aux_min=$am $(python -c "import json;d=json.load(open('gpurun_out/bench_am$am.json'));print(d['ms_per_step'], d['e2e']['value'], d['host_ms_per_step'], d['rounds_per_step'])")"
done
for cfg in "5 32 32" "4 48 32" "4 32 64" "6 32 32"; do set -- $cfg
  ISYCOS_BU_DEPTH=$1 ISYCOS_LOOKAHEAD=$2 ISYCOS_TREND_DEPTH=$3 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sweep > gpurun_out/bench_s.json 2>/dev/null
  echo "D=$1 LA=$2 T=$3 $(python -c "import json;d=json.load(open('gpurun_out/bench_s.json'));print(d['ms_per_step'], d['e2e']['value'], d['host_ms_per_step'], d['rounds_per_step'])")"
done
