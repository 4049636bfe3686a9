#!/bin/bash
# 2-GPU check of the single-launch path for distributed matrices under 2 slices/SM:
# dist parity tests, per-level SpMV times (p2p and NCCL), weak-scaled bench.
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/sm_dist.log 2>&1; echo dist_tests=$?
timeout 300 $TR --master-port 29511 tools/dist_levels.py --grid 161 > gpurun_out/sm_levels.log 2>&1; echo levels=$?
AMGP_HALO=nccl timeout 300 $TR --master-port 29512 tools/dist_levels.py --grid 161 > gpurun_out/sm_levels_nccl.log 2>&1; echo levels_nccl=$?
timeout 300 $TR --master-port 29513 bench.py --gpus 2 --steps 10 --solve-grid 128 > gpurun_out/sm_bench.log 2>&1; echo bench=$?
