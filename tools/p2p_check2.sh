#!/bin/bash
# 2-GPU check of the p2p transport: parity tests, weak-scaled smoother sweep,
# per-level SpMV / exchange costs, and the weak-scaled solve at 161^3.
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/c2_dist.log 2>&1; echo "dist tests $?"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $TR --master-port 29901 bench.py --gpus 2 --steps 10 --solve-grid 128 > gpurun_out/c2_bench.log 2>&1; echo "bench $?"
timeout 300 $TR --master-port 29902 tools/dist_levels.py --grid 161 > gpurun_out/c2_levels.log 2>&1; echo "levels $?"
