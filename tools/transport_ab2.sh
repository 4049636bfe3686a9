#!/bin/bash
# Interleaved A/B of the p2p transports on 2 GPUs (same box): weak-scaled
# smoother sweep, two rounds each.
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for r in 1 2; do for F in 1 0; do
AMGP_P2P_FUSED=$F timeout 300 $TR --master-port 296$r$F bench.py --gpus 2 --steps 10 --solve-grid 0 > gpurun_out/ab_f${F}_r$r.log 2>&1; echo ab$F$r=$?
done; done
