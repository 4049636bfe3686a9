# per-rank rows / nnz / exchange-free SpMV time of the distributed levels (4 GPUs, config 4)
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29542 tools/dist_levels.py --weak-grid 400 --per-rank > gpurun_out/r2_perrank4.json 2> gpurun_out/r2_perrank4.err; echo "levels $?"
tail -n 5 gpurun_out/r2_perrank4.err
