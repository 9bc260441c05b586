cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r2s_build.log 2>&1
# asynchronous submit thread (default) vs synchronous submit, configs[3] 64 pairs and configs[1]
for A in 1 0 1 0; do
  rm -f /tmp/trd; ISYCOS_ASYNC_SUBMIT=$A ISYCOS_TRACE=/tmp/trd timeout 600 python scripts/measure_full.py cfg4 --pairs 64 --reps 3 > $O/r2s_cfg4_a$A.jsonl 2>&1
  python -c "
import json
for l in open('$O/r2s_cfg4_a$A.jsonl'):
    try: d=json.loads(l)
    except Exception: continue
    print('async $A cfg4 rep', d['rep'], 'ms', round(d['ms']), 'host', round(d['kernel']['host_ms']), 'results', d['results'])
"
  grep "^#" /tmp/trd | tail -2
  ISYCOS_ASYNC_SUBMIT=$A timeout 300 python scripts/time_cfg2.py --reps 4 2>&1 | tail -2 | sed "s/^/async $A cfg2 /"
done
timeout 1500 python -m pytest tests/test_gpu_search.py tests/test_gpu_next3.py tests/test_gpu_fullsize.py -q -x > $O/r2s_tests.log 2>&1; echo "tests rc=$?"; tail -2 $O/r2s_tests.log
timeout 900 python bench.py > $O/r2s_bench.json 2> $O/r2s_bench.err; echo "bench rc=$?"
python -c "
import json
d=json.load(open('$O/r2s_bench.json'))
print('bench', round(d['ms_per_step']), 'ms/step', '%.3g' % d['value'], 'frac', round(d['roofline']['frac'],4), 'e2e %.3g' % d['e2e']['value'])
print('cfg2', round(d['side_configs1_search']['ms_per_step'],2), 'sweep', round(d['side_configs2_sweep']['ms_per_step'],2))
"
timeout 1500 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
  --log-file /tmp/r2s_launches.csv python scripts/measure_full.py cfg4 --pairs 16 > $O/r2s_ncu_launches.log 2>&1; echo "ncu launches rc=$?"
python scripts/ncu_summary.py launches /tmp/r2s_launches.csv $O/r2s_launches_cfg4_16pairs.md
head -24 $O/r2s_launches_cfg4_16pairs.md
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sorted_knn|sort_window|block_sort" -c 3 \
  -o /tmp/r2s_sweep4096 python scripts/kernel_bench.py --only 4096 --reps 1 --target 1e11 > $O/r2s_ncu_sweep.log 2>&1; echo "ncu sweep rc=$?"
python scripts/ncu_summary.py rep /tmp/r2s_sweep4096.ncu-rep $O/r2s_ncu_sweep4096.md
python scripts/ncu_summary.py opcodes /tmp/r2s_sweep4096.ncu-rep sorted_knn $O/r2s_sorted_knn_opcodes.txt
cp profiles/issue.json profiles/traffic.json $O/ 2>/dev/null
python scripts/ncu_summary.py issue /tmp/r2s_sweep4096.ncu-rep sorted_throughput "sorted_knn|sort_window|block_sort" $O/issue.json
python scripts/ncu_summary.py traffic /tmp/r2s_sweep4096.ncu-rep sorted_throughput_4096 "sorted_knn|sort_window|block_sort" $O/traffic.json
head -8 $O/r2s_sorted_knn_opcodes.txt
du -sh $O
