R=$GRAFT_REPO_ROOT
export AMGP_WATCHDOG=60
timeout 80 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 tools/nccl_smoke.py > $R/gpurun_out/r2_h3_a.log 2>&1; echo "smoke $?"
AMGP_HALO=nccl timeout 80 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29562 tools/nccl_smoke.py > $R/gpurun_out/r2_h3_b.log 2>&1; echo "smoke nccl $?"
timeout 80 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29563 tools/dsetup_dist_check.py --grid 32 > $R/gpurun_out/r2_h3_c.log 2>&1; echo "check $?"
env | grep -i nccl > $R/gpurun_out/r2_h3_env.log; df -h /dev/shm >> $R/gpurun_out/r2_h3_env.log
