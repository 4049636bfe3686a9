R=$GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_setup.py tests/test_gpu_concurrency.py -q -x > gpurun_out/r2_sigma_pytest.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/r2_sigma_pytest.log
timeout 300 python tools/level_bench.py --m 128 --reps 30 > gpurun_out/r2_lb_sigma.jsonl 2>&1; echo "lb $?"
timeout 900 python tools/ab_solve.py --m 128 --libs default $R/paper_2407_09848_b200/build/libamgp_nosigma.so --rounds 3
timeout 900 python tools/ab_solve.py --m 256 --libs default $R/paper_2407_09848_b200/build/libamgp_nosigma.so --rounds 2
