# The canonical GPU pass of a round (run through gpurun; every artefact lands in gpurun_out/, summaries are
# copied into profiles/ afterwards):  gpurun --timeout 3600 -- 'bash scripts/gpu_pass.sh <tag>'
#   smoke, all -m gpu tests, the default bench line and the reference (oracle) arm, the ncu launch list of a
#   bench step (--clock-control none), one ncu --set full capture of the configs[2] sweep kernels and one of
#   the configs[3] search kernels, and their summaries (issue / traffic JSON for bench.py's roofline object).
TAG=${1:-pass}
cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/${TAG}_build.log 2>&1
nproc > $O/${TAG}_host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> $O/${TAG}_host.txt
timeout 300 python __graft_entry__.py --smoke > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/${TAG}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/${TAG}_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 $O/${TAG}_gpu_tests.log
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/${TAG}_bench_ref.json 2> $O/${TAG}_bench_ref.err; echo "ref rc=$?"
# launch list of a quarter of the bench step (16 of its 64 pairs, same search; a whole step under ncu exceeds the
# time limit): per-kernel shares of the configs[3] search
timeout 1500 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
  --log-file /tmp/${TAG}_launches.csv python scripts/measure_full.py cfg4 --pairs 16 > $O/${TAG}_ncu_launches.log 2>&1; echo "ncu launches rc=$?"
python scripts/ncu_summary.py launches /tmp/${TAG}_launches.csv $O/${TAG}_launches_cfg4_16pairs.md
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sorted_knn|sort_window|block_sort" -c 3 \
  -o /tmp/${TAG}_sweep4096 python scripts/kernel_bench.py --only 4096 --reps 1 --target 1e11 > $O/${TAG}_ncu_sweep.log 2>&1; echo "ncu sweep rc=$?"
python scripts/ncu_summary.py rep /tmp/${TAG}_sweep4096.ncu-rep $O/${TAG}_ncu_sweep4096.md
# opcode mix of the scan kernel (the .ncu-rep files stay on the box: gpurun copies back <= 64 MiB)
python scripts/ncu_summary.py opcodes /tmp/${TAG}_sweep4096.ncu-rep sorted_knn $O/${TAG}_sorted_knn_opcodes.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"warp_sorted|sorted_knn|sort_window|fused_sorted|ksg_lat|ksg_small|ksg_tile|block_sort" \
  -s 3000 -c 8 -o /tmp/${TAG}_cfg4 python scripts/measure_full.py cfg4 --pairs 16 > $O/${TAG}_ncu_cfg4.log 2>&1; echo "ncu cfg4 rc=$?"
python scripts/ncu_summary.py rep /tmp/${TAG}_cfg4.ncu-rep $O/${TAG}_ncu_cfg4.md
python scripts/ncu_summary.py opcodes /tmp/${TAG}_cfg4.ncu-rep warp_sorted $O/${TAG}_warp_sorted_opcodes.txt
cp profiles/issue.json profiles/traffic.json $O/ 2>/dev/null
python scripts/ncu_summary.py issue /tmp/${TAG}_sweep4096.ncu-rep sorted_throughput "sorted_knn|sort_window|block_sort" $O/issue.json
python scripts/ncu_summary.py issue /tmp/${TAG}_cfg4.ncu-rep sorted_marginal "warp_sorted|sorted_knn|sort_window|fused_sorted|block_sort" $O/issue.json
python scripts/ncu_summary.py issue /tmp/${TAG}_cfg4.ncu-rep brute_force "ksg_lat|ksg_small|ksg_tile" $O/issue.json
python scripts/ncu_summary.py traffic /tmp/${TAG}_sweep4096.ncu-rep sorted_throughput_4096 "sorted_knn|sort_window|block_sort" $O/traffic.json
python scripts/ncu_summary.py traffic /tmp/${TAG}_cfg4.ncu-rep sorted_marginal "warp_sorted|sorted_knn|sort_window|fused_sorted|block_sort" $O/traffic.json
python scripts/ncu_summary.py traffic /tmp/${TAG}_cfg4.ncu-rep brute_force "ksg_lat|ksg_small|ksg_tile" $O/traffic.json
du -sh $O
