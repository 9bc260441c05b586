# N > 1 bench flow, code-path check on ONE GPU (ISYCOS_BENCH_DRYRUN=1: 2 ranks share the GPU, gloo collectives;
# never a scaling number): search_sharded over LPT-sharded pairs, all_gather of result windows, max-over-ranks
# timing and the JSON line; then the reference arm under torchrun (rank 0 alone runs it).
cd $GRAFT_REPO_ROOT
O=gpurun_out
python -c "import paper_2204_09131_b200.build as b; b.build()" > $O/r4a_build.log 2>&1
ISYCOS_BENCH_DRYRUN=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --pairs-per-gpu 16 > $O/r4a_dryrun2.json 2> $O/r4a_dryrun2.err; echo "dryrun rc=$?"
tail -c 1500 $O/r4a_dryrun2.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29534 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 > $O/r4a_ref2.json 2> $O/r4a_ref2.err; echo "ref rc=$?"
tail -c 600 $O/r4a_ref2.json
