# round-2 ncu evidence (1 GPU): launch list of the bench sweep, of the 256^3 solve, and
# the --set full capture of the middle smoother step (the bench's roofline kernel)
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --solve-grid 0 --weak-grid 0"
$B > gpurun_out/r2_ncu_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r02_launches_bench.csv $B > gpurun_out/r2_ncu_a.log 2>&1; echo "launches $?"
python tools/run_solve.py --m 256 --repeat 1 > gpurun_out/r2_ncu_solve_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r02_launches_solve256.csv python tools/run_solve.py --m 256 --repeat 1 > gpurun_out/r2_ncu_b.log 2>&1; echo "solve launches $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:Cheb4Step -s 5 -c 1 \
  -o gpurun_out/r02_prof_mid $B > gpurun_out/r2_ncu_c.log 2>&1; echo "full $?"
