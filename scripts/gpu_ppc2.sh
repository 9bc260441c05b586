cd $GRAFT_REPO_ROOT
for p in 2048 1024; do echo "ppc=$p"; for w in 1024 4096 16384; do ISYCOS_SORTED_PPC=$p timeout 300 python scripts/kernel_bench.py --target 1e11 --only $w 2>&1 | tail -1 | cut -c1-120; done; done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -x --timeout 600 -p no:cacheprovider -k "size_classes or segments or cfg3" > gpurun_out/gpu_p2.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/gpu_p2.log
