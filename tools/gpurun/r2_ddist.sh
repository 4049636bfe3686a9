# distributed device setup parity on 2 GPUs (tools/dsetup_dist_check.py)
export AMGP_SETUP_TRACE=1
for cfg in "--grid 32" "--grid 32 --kind pairwise_matching" "--grid 48 --replicate-below 20000" "--grid 20 --stencil 27"; do
  echo "=== $cfg"
  timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/dsetup_dist_check.py $cfg 2>&1 | grep -v "^\s*File\|^\s*\^\|Traceback\|^  " | tail -40
done
