# final evidence for the multi-GPU lines after the in-kernel pack (4 GPUs): bench N=2/4, config 5 N=4, GPU suite, smoke
timeout 900 python bench.py --gpus 2 > gpurun_out/r2g_bench_n2.log 2>&1; echo "bench2 $?"
timeout 900 python bench.py --gpus 4 > gpurun_out/r2g_bench_n4.log 2>&1; echo "bench4 $?"
timeout 900 python bench.py --solve-only --gpus 4 --solve-scaling strong --weak-grid 512 --solve-stencil 27 --solve-k 3 \
  --solve-family opt_cheb1 > gpurun_out/r2g_cfg5_n4.log 2>&1; echo "cfg5 n4 $?"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2g_pytest_gpu.log 2>&1; echo "pytest $?"
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r2g_smoke.log 2>&1; echo "smoke $?"
