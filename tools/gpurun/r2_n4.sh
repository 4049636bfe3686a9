# config 4 at N=4: repeatability and the halo-load variant
run() { echo "=== $*"; timeout 600 python bench.py --solve-only --gpus 4 "$@" 2>/dev/null | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)['solve']; print(d['m'], 'it', d['iterations'], 'solve_ms %.2f'%(1e3*d['solve_s']), 'setup %.1f'%d['setup_s'], 'frac %.3f'%d['roofline_rank0']['frac'], d['clocks_rank0'])"; }
run
run
AMGP_LIB=$PWD/paper_2407_09848_b200/build/libamgp_halonc.so run
AMGP_HALO=nccl run
run --weak-grid 256
AMGP_LIB=$PWD/paper_2407_09848_b200/build/libamgp_halonc.so run --weak-grid 256
timeout 600 python -m pytest tests/test_gpu_concurrency.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
