#!/bin/bash
# Timing experiment: fused p2p launch variants (FUSED_DIAG builds) on 2 GPUs.
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for v in ${VARIANTS:-"" diag1 diag2 diag3}; do
  lib=paper_2407_09848_b200/libamgp${v:+_$v}.so
  AMGP_LIB=$PWD/$lib timeout 300 $TR --master-port 29600 bench.py --gpus 2 --steps 5 --solve-grid 0 > gpurun_out/fd_$v.log 2>&1; echo "$v $?"
done
AMGP_P2P_FUSED=0 timeout 300 $TR --master-port 29601 bench.py --gpus 2 --steps 5 --solve-grid 0 > gpurun_out/fd_two.log 2>&1; echo two $?
