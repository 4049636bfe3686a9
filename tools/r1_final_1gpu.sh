#!/bin/bash
# Round-1 single-GPU measurements: default bench line, BASELINE configs[4]
# shape solve at 1 GPU with the C oracle CPU solve beside it, ncu launch
# list of the 27-point 256^3 solve.
timeout 600 python bench.py > gpurun_out/f1_bench.log 2>&1; echo "bench $?"
timeout 1200 python bench.py --steps 3 --solve-grid 256 --solve-stencil 27 --solve-k 3 \
  --solve-family opt_cheb1 > gpurun_out/f1_bench27.log 2>&1; echo "bench27 $?"
timeout 600 python tools/run_solve.py --m 256 --stencil 27 --family opt_cheb1 --k 3 --repeat 1 \
  > gpurun_out/f1_solve27.log 2>&1; echo "solve27 $?"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/f1_launches_solve27.csv \
  python tools/run_solve.py --m 256 --stencil 27 --family opt_cheb1 --k 3 --repeat 1 \
  > gpurun_out/f1_ncu27.log 2>&1; echo "ncu $?"
