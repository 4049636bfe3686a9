# round-2 final evidence on one box: the whole GPU suite (multi-GPU cases need >=2 GPUs),
# smoke(), and the ncu --set full capture of the middle smoother step (GPU 0 only)
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu_final.log 2>&1; echo "pytest $?"
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r02_smoke_final.log 2>&1; echo "smoke $?"
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --solve-grid 0 --weak-grid 0"
CUDA_VISIBLE_DEVICES=0 timeout 1200 ncu --set full --clock-control none --import-source on \
  --kernel-name-base demangled -k "regex:Cheb4Step<0, 0, 0>" -s 5 -c 1 \
  -o gpurun_out/r02_prof_mid $B > gpurun_out/r2_ncu_c.log 2>&1; echo "full $?"
