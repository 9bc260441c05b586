cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r2m_build.log 2>&1
# size-class routing of the configs[3] search rounds (64 pairs, one call): latency-mode threshold and the
# warp-per-window sorted kernel's lower bound
run() {
  tag=$1; shift
  env "$@" timeout 600 python scripts/measure_full.py cfg4 --pairs 64 --reps 2 > $O/r2m_$tag.jsonl 2>&1
  python - <<PY
import json
for l in open("$O/r2m_$tag.jsonl"):
    try:
        d = json.loads(l)
    except Exception:
        continue
    k = d["kernel"]
    print("$tag rep", d["rep"], "ms", round(d["ms"]), "host", round(k["host_ms"]), "rounds", k["rounds"])
PY
}
rm -f /tmp/trd; run default ISYCOS_TRACE=/tmp/trd
grep "^#" /tmp/trd > $O/r2m_trace_summary.txt
awk '!/^#/ {c=($4>100000)?"big":(($4>2000)?"mid":"small"); n[c]++; h[c]+=$2; s[c]+=$3; a[c]+=$7; m[c]+=$8; w[c]+=$4} END {for (k in n) print k, n[k], "rounds; windows", w[k], "host-since-submit ms", h[k], "submit ms", s[k], "advance ms", a[k], "assemble ms", m[k]}' /tmp/trd >> $O/r2m_trace_summary.txt
run lat1184 ISYCOS_LAT_WINDOWS=1184
run lat2368 ISYCOS_LAT_WINDOWS=2368
run lat9472 ISYCOS_LAT_WINDOWS=9472
run ws129 ISYCOS_WSORTED_MIN_W=129
run ws257 ISYCOS_WSORTED_MIN_W=257
