R=$GRAFT_REPO_ROOT
run() { timeout 90 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 tools/dsetup_dist_check.py --grid 32 > $R/gpurun_out/r2_hang2_$1.log 2>&1; echo "$1 rc $?"; grep -c '"ok": true' $R/gpurun_out/r2_hang2_$1.log; }
AMGP_LIB=$R/paper_2407_09848_b200/build/libamgp_notls.so run 29551
run 29552
nvidia-smi topo -m > $R/gpurun_out/r2_topo.log 2>&1
