cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r2l_build.log 2>&1
free -g > $O/r2l_mem.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next3.py tests/test_gpu_search.py -x -q > $O/r2l_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/r2l_tests.log
# kernel A/B: merge-network top list + pivot-free y searches (libisycos.so) vs the round-2 base build
for L in base new; do
  LIBV=""; [ $L = base ] && LIBV=$GRAFT_REPO_ROOT/paper_2204_09131_b200/libisycos_base.so
  ISYCOS_LIB=$LIBV timeout 600 python scripts/kernel_bench.py --reps 3 > $O/r2l_kbench_$L.jsonl 2>&1
done
cat > /tmp/sweep_ab.py <<'PY'
import json, os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch, bench, paper_2204_09131_b200 as isy
r = bench.sweep_cfg3(isy, torch.cuda.current_stream(), 3)
print(json.dumps({"ms": r["ms_per_step"], "frac": r["roofline"]["frac"], "share": r["roofline"]["kernel_share_of_step"]}))
PY
for L in base new base new; do
  LIBV=""; [ $L = base ] && LIBV=$GRAFT_REPO_ROOT/paper_2204_09131_b200/libisycos_base.so
  echo "sweep $L $(ISYCOS_LIB=$LIBV timeout 300 python /tmp/sweep_ab.py 2>&1 | tail -1)"
done
# concurrent pairs per search call (ISYCOS_MAX_ACTIVE) on configs[3]: the same pairs in one call
for P in 64 128 256; do
  rm -f /tmp/tr$P; ISYCOS_TRACE=/tmp/tr$P ISYCOS_MAX_ACTIVE=$P timeout 600 python scripts/measure_full.py cfg4 --pairs $P --reps 2 > $O/r2l_cfg4_p$P.jsonl 2>&1
  python - <<PY
import json
for l in open("$O/r2l_cfg4_p$P.jsonl"):
    try:
        d = json.loads(l)
    except Exception:
        continue
    k = d["kernel"]
    print("pairs $P rep", d["rep"], "ms", round(d["ms"]), "ms/pair", round(d["ms"] / $P, 1), "host", round(k["host_ms"]),
          "rounds", k["rounds"], "Tcmp/s", round(d["brute_eq_compares_per_s"] / 1e12, 2))
PY
  grep "^#" /tmp/tr$P >> $O/r2l_trace_summary.txt
  awk '!/^#/ {n[$4>20000?"big":"small"]++; h[$4>20000?"big":"small"]+=$2} END {for (k in n) print "P='$P'", k, n[k], "rounds host ms", h[k]}' /tmp/tr$P >> $O/r2l_trace_summary.txt
done
free -g >> $O/r2l_mem.txt
