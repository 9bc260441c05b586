cd $GRAFT_REPO_ROOT
python -c "import paper_2204_09131_b200.build as b; b.build()" > gpurun_out/r2f_build.log 2>&1
timeout 300 python __graft_entry__.py --smoke > gpurun_out/r2f_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2f_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -k "not cfg4_full_size" > gpurun_out/r2f_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2f_gpu_tests.log
ISYCOS_TRACE=gpurun_out/r2f_trace.txt timeout 300 python scripts/measure_full.py cfg4 --pairs 64 --reps 2 > gpurun_out/r2f_cfg4_64.jsonl 2>&1
ISYCOS_LAT_SPLIT=0 timeout 300 python scripts/measure_full.py cfg4 --pairs 64 --reps 2 > gpurun_out/r2f_cfg4_64_nolat.jsonl 2>&1
for f in gpurun_out/r2f_cfg4*.jsonl; do python -c "
import json
for l in open('$f'):
    try:
        d=json.loads(l)
    except Exception:
        continue
    k=d['kernel']; print('$f', d['rep'], 'ms', round(d['ms']), 'host', round(k['host_ms']), 'rounds', k['rounds'])
"; done
grep -h "^#" gpurun_out/r2f_trace.txt
for tool in memcheck synccheck initcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_workload.py > gpurun_out/r2f_sanitize_$tool.log 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/r2f_sanitize_$tool.log
done
