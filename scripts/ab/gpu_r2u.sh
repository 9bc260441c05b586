cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r2u_build.log 2>&1
# routing of sparse size classes in the configs[3] search and the configs[1] search
run() {
  tag=$1; shift
  env "$@" timeout 600 python scripts/measure_full.py cfg4 --pairs 64 --reps 3 > $O/r2u_$tag.jsonl 2>&1
  c4=$(python -c "
import json
ms=[json.loads(l)['ms'] for l in open('$O/r2u_$tag.jsonl') if l.startswith('{')]
print(round(min(ms[1:])) if len(ms)>1 else ms)
")
  c2=$(env "$@" timeout 300 python scripts/time_cfg2.py --reps 5 2>&1 | python -c "
import json,sys
ms=[json.loads(l)['ms'] for l in sys.stdin if l.startswith('{')]
print(round(min(ms[1:]),2) if len(ms)>1 else ms)
")
  echo "$tag cfg4_ms $c4 cfg2_ms $c2"
}
run default X=1
run keep1 ISYCOS_LAT_KEEP_SMALL_R=1
run keep2 ISYCOS_LAT_KEEP_SMALL_R=2
run keep4 ISYCOS_LAT_KEEP_SMALL_R=4
run nofused ISYCOS_FUSED=0
run fused37k ISYCOS_FUSED_MAX_PTS=37888
run ws129 ISYCOS_WSORTED_MIN_W=129
run lat148 ISYCOS_LAT_WINDOWS=148
run default2 X=1
