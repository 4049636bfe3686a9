#!/bin/bash
# Per-level SpMV costs on 2 GPUs with the halo transfer disabled
# (AMGP_HALO=skip: interior + boundary launches, stale halo) vs p2p vs NCCL:
# separates the launch structure from the communication.
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for H in skip p2p nccl; do
AMGP_HALO=$H timeout 300 $TR --master-port 2991${#H} tools/dist_levels.py --grid 161 > gpurun_out/hs_$H.log 2>&1; echo "$H $?"
done
