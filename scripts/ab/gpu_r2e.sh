cd $GRAFT_REPO_ROOT
python -c "import paper_2204_09131_b200.build as b; b.build()" > gpurun_out/r2e_build.log 2>&1
for la in 32 128 512; do
  ISYCOS_TRACE=gpurun_out/r2e_trace_la$la.txt ISYCOS_LOOKAHEAD=$la timeout 300 python scripts/measure_full.py cfg4 --pairs 64 --reps 2 > gpurun_out/r2e_la$la.jsonl 2>&1
done
for la in 64 256; do
  ISYCOS_LOOKAHEAD=$la timeout 300 python scripts/measure_full.py cfg4 --pairs 64 --reps 2 > gpurun_out/r2e_la$la.jsonl 2>&1
done
for d in 2 8; do
  ISYCOS_LOOKAHEAD=128 ISYCOS_BU_DEPTH=$d timeout 300 python scripts/measure_full.py cfg4 --pairs 64 --reps 2 > gpurun_out/r2e_la128_d$d.jsonl 2>&1
done
ISYCOS_LOOKAHEAD=128 ISYCOS_PIPELINE=0 timeout 300 python scripts/measure_full.py cfg4 --pairs 64 --reps 2 > gpurun_out/r2e_la128_nopipe.jsonl 2>&1
ISYCOS_LOOKAHEAD=128 ISYCOS_BLOCK_SORT=0 timeout 300 python scripts/measure_full.py cfg4 --pairs 64 --reps 2 > gpurun_out/r2e_la128_noblock.jsonl 2>&1
ISYCOS_LOOKAHEAD=128 ISYCOS_LAT_WINDOWS=64 timeout 300 python scripts/measure_full.py cfg4 --pairs 64 --reps 2 > gpurun_out/r2e_la128_lat64.jsonl 2>&1
for f in gpurun_out/r2e_*.jsonl; do python -c "
import json
for l in open('$f'):
    try:
        d=json.loads(l)
    except Exception:
        continue
    k=d['kernel']; print('$f', d['rep'], 'ms', round(d['ms']), 'host', round(k['host_ms']), 'rounds', k['rounds'], 'windows', k['windows'], 'distinct', d['stats']['distinct_windows'])
"; done
grep -h "^#" gpurun_out/r2e_trace_*.txt
