cd $GRAFT_REPO_ROOT
rm -f gpurun_out/trace.txt; ISYCOS_TRACE=gpurun_out/trace.txt timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sweep > /dev/null 2>&1; grep "#" gpurun_out/trace.txt | tail -2
rm -f gpurun_out/trace_np.txt; ISYCOS_PIPELINE=0 ISYCOS_TRACE=gpurun_out/trace_np.txt timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sweep > /dev/null 2>&1; grep "#" gpurun_out/trace_np.txt | tail -1
