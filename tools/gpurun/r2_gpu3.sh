# 1 GPU: parity + setup suites, bench default line
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_setup.py -q -x > gpurun_out/r2_pytest3.log 2>&1; echo "pytest $?"
timeout 900 python bench.py > gpurun_out/r2_bench3.log 2>&1; echo "bench $?"
