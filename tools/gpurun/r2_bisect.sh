R=$GRAFT_REPO_ROOT
export AMGP_WATCHDOG=300
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 tools/dsetup_dist_check.py --grid 32 > $R/gpurun_out/r2_bi_check.log 2>&1; echo "check $?"; grep -c '"ok": true' $R/gpurun_out/r2_bi_check.log
timeout 300 python -m pytest tests/test_gpu_concurrency.py -q -x > $R/gpurun_out/r2_bi_conc.log 2>&1; echo "conc $?"
run() { echo "=== $PWD $*"; timeout 400 python bench.py --solve-only "$@" 2>$R/gpurun_out/r2_bi_err.log | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)['solve']; print(d['m'], 'it', d['iterations'], 'solve_ms %.2f'%(1e3*d['solve_s']), 'setup %.1f'%d['setup_s'], 'frac %.3f'%d['roofline_rank0']['frac'])"; }
run --gpus 1
run --gpus 2
cd $R/build_old
run --gpus 1
run --gpus 2
