#!/bin/bash
# 2-GPU: parity tests + per-level SpMV costs (skip / p2p) + weak-scaled sweep.
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/hg_dist.log 2>&1; echo "dist tests $?"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for H in skip p2p; do
AMGP_HALO=$H timeout 300 $TR --master-port 2992${#H} tools/dist_levels.py --grid 161 > gpurun_out/hg_$H.log 2>&1; echo "$H $?"
done
timeout 300 $TR --master-port 29931 bench.py --gpus 2 --steps 10 --solve-grid 128 > gpurun_out/hg_bench.log 2>&1; echo "bench $?"
