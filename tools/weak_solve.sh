#!/bin/bash
# Weak scaling of the PCG + AMG solve at ~256^3 rows per GPU (opt_cheb4 k=4,
# tol 1e-6): 1 GPU 256^3, 2 GPUs 323^3, 4 GPUs 406^3.  Run on a 4-GPU box.
set -x
out=${1:-gpurun_out/weak_solve.log}
CUDA_VISIBLE_DEVICES=0 python tools/run_solve.py --m 256 --family opt_cheb4 --repeat 3 >> $out 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29531 tools/dist_solve.py --grid 323 \
  --replicate-below 20000 120000 --graph 1 >> $out 2>&1
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
  --master-addr 127.0.0.1 --master-port 29532 tools/dist_solve.py --grid 406 \
  --replicate-below 20000 200000 --graph 1 >> $out 2>&1
