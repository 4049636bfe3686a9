# halo gathers: weak L1-cached ld.global (default) vs the L2-only .cg load (AMGP_HALO_LD_CG variant), 4 GPUs
export AMGP_WATCHDOG=600
timeout 900 python -m pytest tests/test_gpu_dist.py -q -x -p no:cacheprovider > gpurun_out/r2_ldca_pytest.log 2>&1; echo "dist tests $?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 \
  tools/p2p_stress.py --iters 4000 > gpurun_out/r2_ldca_stress.log 2>&1; echo "stress $?"
for v in ca cg; do
  if [ $v = cg ]; then export AMGP_LIB=$PWD/paper_2407_09848_b200/libamgp_cg.so; fi
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29542 tools/dist_levels.py --weak-grid 400 > gpurun_out/r2_ldca_dl4_$v.json 2>/dev/null; echo "levels $v $?"
  timeout 600 python bench.py --gpus 4 --steps 10 --warmup 3 --solve-grid 0 --weak-grid 0 --no-cpu-baseline \
    > gpurun_out/r2_ldca_bench4_$v.log 2>&1; echo "bench $v $?"
done
