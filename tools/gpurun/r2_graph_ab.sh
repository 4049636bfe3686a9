# distributed V-cycle: CUDA-graph replay vs eager launches (4 GPUs), weak 256^3 and 400^3 rows/GPU
for g in 256 400; do for dg in 1 0; do
  echo "=== weak $g graph $dg"
  timeout 900 python bench.py --gpus 4 --solve-only --weak-grid $g --dist-graph $dg 2>&1 | grep solve_only | \
    python -c "import json,sys; d=json.loads(sys.stdin.read())['solve']; print(d['m'], d['iterations'], round(d['solve_s']*1e3,2), 'ms', round(d['roofline_rank0']['frac'],3), 'setup', round(d['setup_s'],1))"
done; done
