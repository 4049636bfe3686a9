# BASELINE configs[3] (7-pt 400^3 rows/GPU, opt_cheb4 k=4, weak) and configs[4]
# (27-pt 512^3, opt_cheb1 k=3, strong) at their configured sizes, 1/2/4 GPUs
export AMGP_SETUP_TRACE=1
run() { echo "=== $*"; timeout 900 python bench.py --solve-only "$@" 2>gpurun_out/r2_s4_err.log | grep '^{'; tail -3 gpurun_out/r2_s4_err.log; }
run --gpus 4
run --gpus 4 --solve-scaling strong --weak-grid 512 --solve-stencil 27 --solve-k 3 --solve-family opt_cheb1
run --gpus 2 --solve-scaling strong --weak-grid 512 --solve-stencil 27 --solve-k 3 --solve-family opt_cheb1
run --gpus 1 --solve-scaling strong --weak-grid 512 --solve-stencil 27 --solve-k 3 --solve-family opt_cheb1
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
