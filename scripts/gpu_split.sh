cd $GRAFT_REPO_ROOT
for w in 512 1024 4096; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"sort_window|sorted_knn|rank_merge" --csv --log-file gpurun_out/split_$w.csv python scripts/kernel_bench.py --only $w --reps 1 --target 1e11 > /dev/null 2>&1; echo "w=$w rc=$?"
python - "$w" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(f"gpurun_out/split_{sys.argv[1]}.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
agg = collections.defaultdict(list)
for r in rows[1:]:
    v = float(r[vi].replace(",", "")); u = r[ui]
    v = v / 1e3 if u in ("nsecond", "ns") else v * 1e3 if u in ("msecond", "ms") else v
    agg[r[ki].split("(")[0][:40]].append(v)
for k, v in agg.items(): print(k, len(v), "median us", sorted(v)[len(v)//2])
PY
done
