# NVLink ordered all-reduce for the PCG dots (AMGP_P2P_ALLREDUCE): multi-GPU parity, then 128^3/GPU weak solve A/B (4 GPUs)
export AMGP_WATCHDOG=900
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -x -p no:cacheprovider > gpurun_out/r2_red_pytest.log 2>&1; echo "dist tests $?"
tail -1 gpurun_out/r2_red_pytest.log
for ar in 1 0 1 0; do
  AMGP_P2P_ALLREDUCE=$ar timeout 600 python bench.py --solve-only --weak-grid 128 --gpus 4 > gpurun_out/r2_red_w128_$ar.log 2>&1
  echo "ar=$ar $(grep solve_only gpurun_out/r2_red_w128_$ar.log | python -c "import json,sys; d=json.loads(sys.stdin.read())['solve']; print(d['iterations'], d['final_relres'], round(d['solve_s']*1e3,2))")"
done
