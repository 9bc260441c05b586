cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r2x_build.log 2>&1
cat > /tmp/sweep_once.py <<'PY'
import json, os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch, bench, paper_2204_09131_b200 as isy
r = bench.sweep_cfg3(isy, torch.cuda.current_stream(), 1)
print(json.dumps({"ms": r["ms_per_step"]}))
PY
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file /tmp/r2x_sweep.csv python /tmp/sweep_once.py > /dev/null 2>&1; echo "ncu sweep rc=$?"
python scripts/ncu_summary.py launches /tmp/r2x_sweep.csv $O/r2x_launches_sweep.md; head -14 $O/r2x_launches_sweep.md
python - <<'PY'
import csv
rows = list(csv.reader(open('/tmp/r2x_sweep.csv')))
hdr = [r for r in rows if 'Kernel Name' in r][0]
ik, iv, im, ig = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Name'), hdr.index('ID')
seq = []
for r in rows:
    if len(r) > iv and r[im] == 'gpu__time_duration.sum':
        seq.append((r[ik].split('(')[0].split('::')[-1][:40], r[iv]))
print('launch sequence (kernel, duration):')
for k, v in seq[:80]: print(' ', k, v)
PY
