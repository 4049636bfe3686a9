# fused interior+boundary launch (p2p halo): correctness, stress, then A/B vs two launches (4 GPUs)
export AMGP_WATCHDOG=600
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -p no:cacheprovider > gpurun_out/r2_fuse_pytest.log 2>&1; echo "dist tests $?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 \
  tools/p2p_stress.py --iters 4000 > gpurun_out/r2_fuse_stress.log 2>&1; echo "stress $?"
for fz in 1 0; do
  AMGP_HALO_FUSE=$fz timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29542 tools/dist_levels.py --weak-grid 400 > gpurun_out/r2_fuse_dl4_$fz.json 2>/dev/null; echo "levels fuse=$fz $?"
  AMGP_HALO_FUSE=$fz timeout 600 python bench.py --gpus 4 --steps 10 --warmup 3 --solve-grid 0 --weak-grid 0 --no-cpu-baseline \
    > gpurun_out/r2_fuse_bench4_$fz.log 2>&1; echo "bench fuse=$fz $?"
done
