#!/bin/bash
# A/B of the p2p halo transports on 2 GPUs: dist parity tests, weak-scaled
# smoother sweep, per-level SpMV + exchange times (AMGP_P2P_FUSED=0: pack
# kernel + boundary launch; 1: one fused launch, the default).
set -x
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
free -g | head -2; nproc
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/t2_dist.log 2>&1; echo dist_tests=$?
for F in 0 1; do
AMGP_P2P_FUSED=$F timeout 300 $TR --master-port 2950$F bench.py --gpus 2 --steps 10 --solve-grid 128 > gpurun_out/t2_bench_f$F.log 2>&1; echo bench$F=$?
AMGP_P2P_FUSED=$F timeout 300 $TR --master-port 2951$F tools/dist_levels.py --grid 161 > gpurun_out/t2_levels_f$F.log 2>&1; echo levels$F=$?
done
