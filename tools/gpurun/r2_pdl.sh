# programmatic dependent launch of the single-GPU row kernels: parity, then solve A/B (AMGP_PDL=0/1)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_setup.py tests/test_gpu_concurrency.py -q -x \
  -p no:cacheprovider > gpurun_out/r2_pdl_pytest.log 2>&1; echo "parity $?"; tail -1 gpurun_out/r2_pdl_pytest.log
for m in 64 128 256; do
  echo "== m=$m"; timeout 900 python tools/ab_solve.py --m $m --libs AMGP_PDL=0 AMGP_PDL=1 --rounds 3
done > gpurun_out/r2_pdl_ab.log 2>&1; cat gpurun_out/r2_pdl_ab.log
AMGP_PDL=0 timeout 600 python bench.py --steps 5 --warmup 3 --weak-grid 0 --solve-grid 0 --no-cpu-baseline > gpurun_out/r2_pdl_bench0.log 2>&1
AMGP_PDL=1 timeout 600 python bench.py --steps 5 --warmup 3 --weak-grid 0 --solve-grid 0 --no-cpu-baseline > gpurun_out/r2_pdl_bench1.log 2>&1
for f in 0 1; do tail -1 gpurun_out/r2_pdl_bench$f.log | cut -c1-200; done
