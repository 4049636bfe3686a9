# decomposition of the distributed SpMV overhead (4 GPUs, config 4 levels): with and without the
# exchange protocol (AMGP_HALO_NOSYNC=1: no pack, no waits -- timing only), fused and two launches
for ns in 1 0; do for fz in 1 0; do
  AMGP_HALO_NOSYNC=$ns AMGP_HALO_FUSE=$fz timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port 29542 tools/dist_levels.py --weak-grid 400 --no-solve \
    > gpurun_out/r2_ns${ns}_fz${fz}.json 2>/dev/null; echo "nosync=$ns fuse=$fz $?"
done; done
