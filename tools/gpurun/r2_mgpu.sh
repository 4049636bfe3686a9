# multi-GPU solve efficiency experiments (4 GPUs): config 4 and 256^3 rows/GPU
run() { echo "=== $*"; timeout 600 python bench.py --solve-only "$@" 2>gpurun_out/r2_mgpu_err.log | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)['solve']; print(d['n_gpus'] if 'n_gpus' in d else '', d['m'], d['levels'], 'dist', d['distributed_levels'], 'it', d['iterations'], 'solve_ms %.2f'%(1e3*d['solve_s']), 'setup %.1f'%d['setup_s'], 'frac %.3f'%d['roofline_rank0']['frac'])"; }
run --gpus 1 --weak-grid 256
run --gpus 2 --weak-grid 256
run --gpus 4 --weak-grid 256
run --gpus 4 --weak-grid 256 --krylov pcg1
run --gpus 4 --weak-grid 256 --replicate-below 200000
AMGP_HALO=nccl run --gpus 4 --weak-grid 256
run --gpus 4
run --gpus 4 --krylov pcg1
run --gpus 4 --replicate-below 400000
run --gpus 4 --weak-grid 128
run --gpus 1 --weak-grid 128
