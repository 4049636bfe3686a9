#!/bin/bash
# 4-GPU diagnosis of the 27-point 256^3 strong-scaling point: per-level SpMV
# and exchange costs (slowest rank) and the solve at several coarse-level
# replication thresholds.
C=/tmp/amgp_s27_256
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 1200 $TR --master-port 29801 tools/dist_solve.py --grid 256 --stencil 27 --family opt_cheb1 --k 3 \
  --replicate-below 20000 150000 --graph 1 --repeat 6 --cache $C > gpurun_out/s27_solve.log 2>&1; echo "solve $?"
timeout 1200 $TR --master-port 29802 tools/dist_levels.py --grid 256 --stencil 27 --reps 30 --cache $C \
  > gpurun_out/s27_levels.log 2>&1; echo "levels $?"
