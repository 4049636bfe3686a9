#!/bin/bash
# Quick 2-GPU A/B of the p2p transports (two-launch vs fused): weak-scaled
# smoother sweep and per-level SpMV + exchange times.
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for F in ${FUSED:-0 1}; do
AMGP_P2P_FUSED=$F timeout 300 $TR --master-port 2950$F bench.py --gpus 2 --steps 10 --solve-grid ${SOLVE:-128} > gpurun_out/q_bench_f$F.log 2>&1; echo bench$F=$?
AMGP_P2P_FUSED=$F timeout 300 $TR --master-port 2951$F tools/dist_levels.py --grid 161 > gpurun_out/q_levels_f$F.log 2>&1; echo levels$F=$?
done
