# round-2 final evidence on one 4-GPU box (final code): driver-style bench lines N=1/2/4,
# config 5 at N=4 (fused distributed launch), reference arm, full GPU suite, smoke
timeout 900 python bench.py > gpurun_out/r2f_bench_n1.log 2>&1; echo "bench1 $?"
timeout 900 python bench.py --gpus 2 > gpurun_out/r2f_bench_n2.log 2>&1; echo "bench2 $?"
timeout 900 python bench.py --gpus 4 > gpurun_out/r2f_bench_n4.log 2>&1; echo "bench4 $?"
timeout 900 python bench.py --solve-only --gpus 4 --solve-scaling strong --weak-grid 512 --solve-stencil 27 --solve-k 3 \
  --solve-family opt_cheb1 > gpurun_out/r2f_cfg5_n4.log 2>&1; echo "cfg5 n4 $?"
timeout 600 python bench.py --impl reference > gpurun_out/r2f_ref_n1.log 2>&1; echo "ref $?"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2f_pytest_gpu.log 2>&1; echo "pytest $?"
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r2f_smoke.log 2>&1; echo "smoke $?"
