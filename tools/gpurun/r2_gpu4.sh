# 2 GPUs: new parity/concurrency/drop-in tests, the reference's own suite, p2p stress
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_concurrency.py tests/test_gpu_dropin.py -q -x > gpurun_out/r2_pytest4.log 2>&1; echo "pytest $?"
timeout 900 python tests/test_gpu_dropin.py > gpurun_out/r2_dropin_ref_suite.log 2>&1; echo "dropin $?"
for t in p2p nccl; do
  AMGP_HALO=$t timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 tools/p2p_stress.py --iters 10000 > gpurun_out/r2_stress_$t.log 2>&1; echo "stress $t $?"
done
