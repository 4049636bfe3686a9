# round-2 evidence on 4 GPUs: driver-style bench lines, config 5 at N=2/4
R=$GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/r2_final_bench_n1.log 2>&1; echo "bench1 $?"
timeout 900 python bench.py --gpus 4 > gpurun_out/r2_final_bench_n4.log 2>&1; echo "bench4 $?"
timeout 900 python bench.py --gpus 2 > gpurun_out/r2_final_bench_n2.log 2>&1; echo "bench2 $?"
for n in 4 2; do
timeout 900 python bench.py --solve-only --gpus $n --solve-scaling strong --weak-grid 512 --solve-stencil 27 --solve-k 3 --solve-family opt_cheb1 > gpurun_out/r2_final_cfg5_n$n.log 2>&1; echo "cfg5 n$n $?"
done
timeout 900 python bench.py --impl reference > gpurun_out/r2_final_ref_n1.log 2>&1; echo "ref $?"
