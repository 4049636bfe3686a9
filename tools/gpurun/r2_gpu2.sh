# round-2 GPU check on 2 GPUs: full gpu suite, bench at N=2 (sweep + config-4 weak solve at 504^3)
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2_pytest2.log 2>&1; echo "pytest $?"
timeout 900 python bench.py --gpus 2 > gpurun_out/r2_bench2_n2.log 2>&1; echo "bench2 $?"
