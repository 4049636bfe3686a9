#!/bin/bash
# Strong scaling of the PCG + AMG solve (BASELINE configs[4] shape: 27-point
# stencil, opt_cheb1 k = 3, rtol 1e-6) on 1 / 2 / 4 GPUs of one box.  The
# hierarchy is built once (native host setup, rank 0) and cached on local
# disk for the three world sizes.  GRID (default 256), STENCIL (default 27).
G=${GRID:-256}; S=${STENCIL:-27}; F=${FAMILY:-opt_cheb1}; K=${DEGREE:-3}
out=${1:-gpurun_out/strong_solve.log}
CACHE=${CACHE:-/tmp/amgp_strong_${S}_${G}}
nproc; free -g | head -2; df -h /tmp | tail -1
for W in 1 2 4; do
  timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $W --master-addr 127.0.0.1 \
    --master-port 2970$W tools/dist_solve.py --grid $G --stencil $S --family $F --k $K \
    --replicate-below 20000 --graph 1 --repeat 3 --cache $CACHE >> $out 2>&1
  echo "world $W: $?"
done
