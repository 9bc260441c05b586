cd $GRAFT_REPO_ROOT
for p in 1024 512 256; do echo "ppc=$p"; for w in 1024 4096 16384; do ISYCOS_SORTED_PPC=$p timeout 300 python scripts/kernel_bench.py --target 1e11 --only $w 2>&1 | tail -1 | cut -c1-120; done; done
