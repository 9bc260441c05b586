cd $GRAFT_REPO_ROOT
for mw in 257 513 1025 2049 4097; do
  ISYCOS_SORTED_MIN_W=$mw timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_minw_$mw.json 2>/dev/null
  echo "minw=$mw $(python -c "import json;d=json.load(open('gpurun_out/bench_minw_$mw.json'));print(d['ms_per_step'], d['host_ms_per_step'], d['rounds_per_step'], d['roofline']['paths'])")"
done
