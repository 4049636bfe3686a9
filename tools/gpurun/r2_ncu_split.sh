# ncu of the split-slice schedule on the 128^3 level-2 matrix (+ per-level eager timings)
timeout 300 python tools/level_bench.py --m 128 --reps 30 > gpurun_out/r2_levels2.jsonl 2>&1; echo "lb $?"
timeout 300 python tools/run_solve.py --m 128 --repeat 1 > gpurun_out/r2_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_split_rows -c 3 -o gpurun_out/r2_split \
  python tools/run_solve.py --m 128 --repeat 1 > gpurun_out/r2_ncu_split.log 2>&1; echo "ncu $?"
