#!/bin/bash
# 4-GPU box: dist parity tests (2 and 4 ranks, both launch structures) and
# the default bench at N = 2 and 4 as the driver launches it.
timeout 1200 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/g4_dist.log 2>&1; echo "dist tests $?"
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 2980$N bench.py --gpus $N > gpurun_out/g4_bench_n$N.log 2>&1; echo "bench n$N $?"
done
