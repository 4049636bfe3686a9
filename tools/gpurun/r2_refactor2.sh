# refactor check of the distributed launch path on 2 GPUs: multi-GPU parity tests (2-GPU cases), stress
export AMGP_WATCHDOG=900
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -p no:cacheprovider -rs > gpurun_out/r2_ref2_pytest.log 2>&1; echo "dist tests $?"
tail -3 gpurun_out/r2_ref2_pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 \
  tools/p2p_stress.py --iters 3000 > gpurun_out/r2_ref2_stress.log 2>&1; echo "stress $?"
grep -c '"ok": true' gpurun_out/r2_ref2_stress.log
