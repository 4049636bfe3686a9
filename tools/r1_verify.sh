nvidia-smi --query-gpu=name --format=csv,noheader | head -1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v_pytest.log 2>&1; echo "pytest $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v_smoke.log 2>&1; echo "smoke $?"
timeout 600 python bench.py > gpurun_out/v_bench.log 2>&1; echo "bench $?"
timeout 600 python bench.py --impl reference > gpurun_out/v_bench_ref.log 2>&1; echo "ref $?"
