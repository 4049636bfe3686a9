# coarse-row rebalancing of the distributed setup: parity tests, stress, per-level timing, configs 4/5 (4 GPUs)
export AMGP_WATCHDOG=900
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -x -p no:cacheprovider > gpurun_out/r2_rebal_pytest.log 2>&1; echo "dist tests $?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 \
  tools/p2p_stress.py --iters 3000 > gpurun_out/r2_rebal_stress.log 2>&1; echo "stress $?"
AMGP_SETUP_TRACE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29542 tools/dist_levels.py --weak-grid 400 --per-rank > gpurun_out/r2_rebal_dl4.json 2> gpurun_out/r2_rebal_dl4.err; echo "levels $?"
timeout 900 python bench.py --gpus 4 --solve-only --weak-grid 400 > gpurun_out/r2_rebal_cfg4_n4.log 2>&1; echo "cfg4 n4 $?"
timeout 900 python bench.py --gpus 2 --solve-only --weak-grid 400 > gpurun_out/r2_rebal_cfg4_n2.log 2>&1; echo "cfg4 n2 $?"
timeout 900 python bench.py --solve-only --gpus 4 --solve-scaling strong --weak-grid 512 --solve-stencil 27 --solve-k 3 \
  --solve-family opt_cheb1 > gpurun_out/r2_rebal_cfg5_n4.log 2>&1; echo "cfg5 n4 $?"
