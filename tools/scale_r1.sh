#!/bin/bash
# Round-1 scaling runs on one 4-GPU box: dist parity tests, strong scaling
# (27-point 256^3, opt_cheb1 k=3), weak scaling at 400^3 rows per GPU
# (BASELINE configs[3]: opt_cheb4 k=4; 1 GPU 400^3, 2 GPUs 504^3 -- 635^3 on
# 4 GPUs needs ~470 GB of host memory for the host setup and is not run).
out=gpurun_out/scale_r1.log
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/scale_tests.log 2>&1; echo "dist tests: $?"
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
C27=/tmp/amgp_s27_256
for W in 1 2 4; do
  timeout 1800 $TR --nproc-per-node $W --master-port 2971$W tools/dist_solve.py --grid 256 --stencil 27 \
    --family opt_cheb1 --k 3 --replicate-below 20000 --graph 1 --repeat 8 --cache $C27 >> $out 2>&1
  echo "strong world $W: $?"
done
rm -rf $C27
timeout 1800 $TR --nproc-per-node 1 --master-port 29721 tools/dist_solve.py --grid 400 --family opt_cheb4 --k 4 \
  --replicate-below 20000 --graph 1 --repeat 5 >> $out 2>&1; echo "weak 1: $?"
timeout 2400 $TR --nproc-per-node 2 --master-port 29722 tools/dist_solve.py --grid 504 --family opt_cheb4 --k 4 \
  --replicate-below 20000 --graph 1 --repeat 5 >> $out 2>&1; echo "weak 2: $?"
