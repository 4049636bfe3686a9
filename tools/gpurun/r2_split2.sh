R=$GRAFT_REPO_ROOT
timeout 300 python tools/level_bench.py --m 128 --reps 30 > gpurun_out/r2_lb_new.jsonl 2>&1; echo "new $?"
AMGP_LIB=$R/paper_2407_09848_b200/build/libamgp_u8.so timeout 300 python tools/level_bench.py --m 128 --reps 30 > gpurun_out/r2_lb_u8.jsonl 2>&1; echo "u8 $?"
timeout 300 python tools/level_bench.py --m 256 --reps 10 > gpurun_out/r2_lb_new256.jsonl 2>&1; echo "new256 $?"
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_setup.py -q -x > gpurun_out/r2_split2_pytest.log 2>&1; echo "pytest $?"; tail -1 gpurun_out/r2_split2_pytest.log
