# ncu --set full of the middle cheb4 smoother step (the bench's roofline kernel), GPU 0
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --solve-grid 0 --weak-grid 0"
timeout 1200 ncu --set full --clock-control none --import-source on \
  --kernel-name-base demangled -k "regex:Cheb4Step<.bool.0, .bool.0, .bool.0>" -s 5 -c 1 \
  -o gpurun_out/r02_prof_mid $B > gpurun_out/r2_ncu_c.log 2>&1; echo "full $?"
