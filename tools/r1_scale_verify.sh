#!/bin/bash
# driver-style scaling launches of the default bench at N = 2 and 4 (+ reference arm)
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29$((500+N)) bench.py --gpus $N --steps 20 --warmup 3 > gpurun_out/s_bench_n$N.log 2>&1; echo "bench n$N $?"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --impl reference --gpus 2 --steps 20 --warmup 3 > gpurun_out/s_ref_n2.log 2>&1; echo "ref n2 $?"
