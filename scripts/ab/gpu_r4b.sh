# ksg_lat register allocation A/B: default bounds (44 registers, 5 CTAs/SM) vs ISY_LAT_MINB=3 (76 registers, no
# rematerialisation pressure) vs ISY_LAT_MINB=6 (40 registers, 8 B of spills, 6 CTAs/SM); alternative libraries
# built beforehand (build(defines, out)), loaded through ISYCOS_LIB
cd $GRAFT_REPO_ROOT
O=gpurun_out
P=paper_2204_09131_b200
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r4b_build.log 2>&1
for V in minb3 minb6; do
  ISYCOS_LIB=$PWD/$P/libisycos_$V.so timeout 900 python -m pytest tests/test_gpu_next3.py tests/test_gpu_search.py -q -x > $O/r4b_tests_$V.log 2>&1; echo "tests $V rc=$?"; tail -1 $O/r4b_tests_$V.log
done
for V in base minb3 minb6 base minb3 minb6; do
  L=$PWD/$P/libisycos_$V.so; [ $V = base ] && L=$PWD/$P/libisycos.so
  c4=$(ISYCOS_LIB=$L timeout 600 python scripts/measure_full.py cfg4 --pairs 64 --reps 3 2>&1 | python -c "
import json,sys
print([round(json.loads(l)['ms']) for l in sys.stdin if l.startswith('{')][1:])
")
  c2=$(ISYCOS_LIB=$L timeout 300 python scripts/time_cfg2.py --reps 5 2>&1 | python -c "
import json,sys
print([round(json.loads(l)['ms'],1) for l in sys.stdin if l.startswith('{')][1:])
")
  echo "$V cfg4 $c4 cfg2 $c2"
done
