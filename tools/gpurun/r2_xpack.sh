# halo pack inside the fused row kernel (AMGP_HALO_XPACK): parity, stress, per-level timing, sweep and config 4 (4 GPUs)
export AMGP_WATCHDOG=900
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -x -p no:cacheprovider > gpurun_out/r2_xpack_pytest.log 2>&1; echo "dist tests $?"
AMGP_HALO_FUSE=2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29541 tools/p2p_stress.py --iters 3000 > gpurun_out/r2_xpack_stress.log 2>&1; echo "stress fuse2 $?"
for cfg in "1 1" "2 1" "1 0"; do set -- $cfg
  AMGP_HALO_FUSE=$1 AMGP_HALO_XPACK=$2 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port 29542 tools/dist_levels.py --weak-grid 400 --no-solve \
    > gpurun_out/r2_xpack_dl_$1$2.json 2>/dev/null; echo "levels fuse=$1 xpack=$2 $?"
  AMGP_HALO_FUSE=$1 AMGP_HALO_XPACK=$2 timeout 600 python bench.py --gpus 4 --steps 10 --warmup 3 --solve-grid 0 \
    --no-cpu-baseline > gpurun_out/r2_xpack_bench4_$1$2.log 2>&1; echo "bench fuse=$1 xpack=$2 $?"
done
