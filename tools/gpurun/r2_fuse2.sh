# heuristic fused launch (AMGP_HALO_FUSE=1 default): levels, sweep and config-4 solve at 4 GPUs
export AMGP_WATCHDOG=600
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29542 tools/dist_levels.py --weak-grid 400 > gpurun_out/r2_fuse_dl4_h.json 2>/dev/null; echo "levels $?"
timeout 600 python bench.py --gpus 4 --steps 10 --warmup 3 --solve-grid 0 --weak-grid 0 --no-cpu-baseline \
    > gpurun_out/r2_fuse_bench4_h.log 2>&1; echo "bench $?"
timeout 900 python bench.py --gpus 4 --solve-only --weak-grid 400 > gpurun_out/r2_fuse_solve4_h.log 2>&1; echo "solve $?"
timeout 900 python bench.py --gpus 2 --solve-only --weak-grid 400 > gpurun_out/r2_fuse_solve2_h.log 2>&1; echo "solve2 $?"
