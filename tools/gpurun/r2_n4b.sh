# config 4 at N=4: HEAD vs the r2_scale4 code (worktree build_old), allocator setting
R=$GRAFT_REPO_ROOT
run() { echo "=== $PWD $*"; timeout 600 python bench.py --solve-only --gpus 4 "$@" 2>$R/gpurun_out/r2_n4b_err.log | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)['solve']; print(d['m'], 'it', d['iterations'], 'solve_ms %.2f'%(1e3*d['solve_s']), 'setup %.1f'%d['setup_s'], 'frac %.3f'%d['roofline_rank0']['frac'])"; tail -2 $R/gpurun_out/r2_n4b_err.log | grep -v OMP; }
cd $R/build_old
PYTORCH_CUDA_ALLOC_CONF=expandable_segments:False run
run
cd $R
run
timeout 600 python -m pytest tests/test_gpu_concurrency.py -q -x > gpurun_out/r2_conc.log 2>&1; tail -2 gpurun_out/r2_conc.log
