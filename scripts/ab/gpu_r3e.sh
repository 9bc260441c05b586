# sorted_knn (throughput scan) memory-pipe breakdown: is the scan bound by L1 wavefronts of its scattered LDGs?
cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r3e_build.log 2>&1
for W in 16384 4096; do
timeout 600 ncu --set full --clock-control none -k regex:"sorted_knn" -c 1 -o /tmp/r3e_$W \
  python scripts/kernel_bench.py --only $W --reps 1 --target 1e11 > $O/r3e_ncu_$W.log 2>&1; echo "ncu $W rc=$?"
ncu -i /tmp/r3e_$W.ncu-rep --page details --print-details all > $O/r3e_details_$W.txt 2>&1
ncu -i /tmp/r3e_$W.ncu-rep --page raw --csv > /tmp/r3e_raw_$W.csv 2>&1
python - <<PY > $O/r3e_l1_$W.txt
import csv
rows=list(csv.reader(open('/tmp/r3e_raw_$W.csv')))
h=rows[0]; v=rows[2] if len(rows)>2 else rows[1]
for a,b in zip(h,v):
    if any(t in a for t in ('l1tex__t_','l1tex__data','l1tex__lsu','lsu_mem_global','l1tex__throughput','l1tex__m_','smsp__inst_executed_op_global','smsp__sass_inst_executed_op_global','sm__memory_throughput','l1tex__f_')):
        print(a,b)
PY
done
