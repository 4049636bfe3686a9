# BASELINE configs[4] (27-pt 512^3, opt_cheb1 k=3, strong) on 2 and 1 GPUs
export AMGP_SETUP_TRACE=1
for n in 2 1; do
  echo "=== gpus $n"
  timeout 900 python bench.py --solve-only --gpus $n --solve-scaling strong --weak-grid 512 --solve-stencil 27 --solve-k 3 --solve-family opt_cheb1 > gpurun_out/r2_s5_out$n.log 2> gpurun_out/r2_s5_err$n.log
  echo "rc $?"; grep '^{' gpurun_out/r2_s5_out$n.log; grep -v "^\[rank\|amgp setup" gpurun_out/r2_s5_err$n.log | tail -12
done
