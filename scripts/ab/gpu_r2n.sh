cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r2n_build.log 2>&1
B=$GRAFT_REPO_ROOT/paper_2204_09131_b200/libisycos_b.so
# A/B: unconditional block merge in phase A (ISY_MERGE_ALWAYS, libisycos_b.so) vs the guarded merge
cat > /tmp/sweep_ab.py <<'PY'
import json, os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import torch, bench, paper_2204_09131_b200 as isy
r = bench.sweep_cfg3(isy, torch.cuda.current_stream(), 3)
print(json.dumps({"ms": r["ms_per_step"], "frac": r["roofline"]["frac"]}))
PY
for L in a b a b; do
  LIBV=""; [ $L = b ] && LIBV=$B
  echo "sweep $L $(ISYCOS_LIB=$LIBV timeout 300 python /tmp/sweep_ab.py 2>&1 | tail -1)"
done
for L in a b; do
  LIBV=""; [ $L = b ] && LIBV=$B
  for W in 128 512 4096 16384; do
    ISYCOS_LIB=$LIBV timeout 300 python scripts/kernel_bench.py --only $W --reps 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kbench $L', d['w'], round(d['kernel_ms'],3))"
  done
done
run() {
  tag=$1; shift
  env "$@" timeout 600 python scripts/measure_full.py cfg4 --pairs 64 --reps 2 > $O/r2n_$tag.jsonl 2>&1
  python - <<PY
import json
for l in open("$O/r2n_$tag.jsonl"):
    try:
        d = json.loads(l)
    except Exception:
        continue
    k = d["kernel"]
    print("$tag rep", d["rep"], "ms", round(d["ms"]), "host", round(k["host_ms"]), "rounds", k["rounds"])
PY
}
run cfg4_a X=1
run cfg4_b ISYCOS_LIB=$B
run cfg4_aux2k ISYCOS_AUX_MIN_WINDOWS=2048
run cfg4_noaux ISYCOS_AUX_MIN_WINDOWS=1000000000
