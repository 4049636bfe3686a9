# TEMPORARY timing experiment (results wrong in modes 2/3): what makes the fused launch slow on the fine level
for dbg in 0 2 3; do
  AMGP_HALO_FUSE=2 AMGP_FUSE_DBG=$dbg timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port 29542 tools/dist_levels.py --weak-grid 400 --no-solve \
    > gpurun_out/r2_fusedbg_$dbg.json 2>/dev/null; echo "dbg=$dbg $?"
done
