# 4 GPUs: whole gpu suite + driver-style bench at N=4 and N=2
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_pytest5.log 2>&1; echo "pytest $?"
timeout 900 python bench.py --gpus 4 > gpurun_out/r2_bench5_n4.log 2>&1; echo "bench4 $?"
timeout 900 python bench.py --gpus 2 > gpurun_out/r2_bench5_n2.log 2>&1; echo "bench2 $?"
