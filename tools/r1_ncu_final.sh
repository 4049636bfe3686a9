#!/bin/bash
# Launch list of the default bench command, then one --set full capture of a
# cheb4 middle degree step (256^3) from the same bench.
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --solve-grid 0 > gpurun_out/n_bench.log 2>&1; echo "bench $?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/n_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --solve-grid 0 \
  > gpurun_out/n_ncu_list.log 2>&1; echo "ncu list $?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:_Z13k_thread_rowsI9Cheb4StepILb0ELb0ELb0EE --launch-skip 10 -c 1 -o gpurun_out/r01_mid_full \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --solve-grid 0 > gpurun_out/n_ncu_full.log 2>&1; echo "ncu full $?"
