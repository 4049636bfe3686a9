# per-level SpMV times of the weak-scaled hierarchy at 1, 2 and 4 GPUs (400^3 rows per GPU)
timeout 600 python tools/dist_levels.py --weak-grid 400 > gpurun_out/r2_dl_1.json 2> gpurun_out/r2_dl_1.err
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533 \
  tools/dist_levels.py --weak-grid 400 > gpurun_out/r2_dl_$n.json 2> gpurun_out/r2_dl_$n.err
done
tail -n 3 gpurun_out/r2_dl_*.err
