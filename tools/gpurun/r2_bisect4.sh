R=$GRAFT_REPO_ROOT
export AMGP_WATCHDOG=500
run() { echo "=== $PWD $AMGP_LIB $*"; timeout 500 python bench.py --solve-only --gpus 4 "$@" 2>$R/gpurun_out/r2_bi4_err.log | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)['solve']; print(d['m'], 'it', d['iterations'], 'solve_ms %.2f'%(1e3*d['solve_s']), 'setup %.1f'%d['setup_s'], 'frac %.3f'%d['roofline_rank0']['frac'])"; }
cd $R; run
AMGP_LIB=$R/paper_2407_09848_b200/build/libamgp_stride32.so run
unset AMGP_LIB
cd $R/build_6675f07; run
cd $R/build_943679e; run
cd $R/build_old; run
