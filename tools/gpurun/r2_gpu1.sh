# round-2 GPU check: full gpu suite, default bench line
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest1.log 2>&1; echo "pytest $?"
timeout 900 python bench.py > gpurun_out/r2_bench1.log 2>&1; echo "bench $?"
