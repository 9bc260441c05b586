cd $GRAFT_REPO_ROOT
for f in 0 1000000000; do echo "fused_max_pts=$f"; for w in 512 1024 4096; do ISYCOS_FUSED_MAX_PTS=$f timeout 300 python scripts/kernel_bench.py --target 1e11 --only $w 2>&1 | tail -1 | cut -c1-110; done; done
