R=$GRAFT_REPO_ROOT
export AMGP_WATCHDOG=500
timeout 500 python bench.py --solve-only --gpus 4 2>/dev/null | grep '^{' > gpurun_out/r2_fix_n4.json; python -c "
import json; d=json.load(open('gpurun_out/r2_fix_n4.json'))['solve']; print(d['m'], d['iterations'], round(1e3*d['solve_s'],2), round(d['setup_s'],1))"
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_concurrency.py -q > gpurun_out/r2_fix_dist.log 2>&1; echo "dist $?"; tail -2 gpurun_out/r2_fix_dist.log
