# weak scaling of the PCG+AMG solve at 256^3 and 128^3 rows per GPU (final code), N = 1, 2, 4
for g in 256 128; do
  timeout 600 python bench.py --solve-only --weak-grid $g > gpurun_out/r2w_${g}_n1.log 2>&1; echo "w$g n1 $?"
  for n in 2 4; do
    timeout 900 python bench.py --solve-only --weak-grid $g --gpus $n > gpurun_out/r2w_${g}_n$n.log 2>&1; echo "w$g n$n $?"
  done
done
for f in gpurun_out/r2w_*.log; do echo "$f $(grep solve_only $f | python -c "import json,sys; d=json.loads(sys.stdin.read())['solve']; print(d['m'], d['iterations'], round(d['solve_s']*1e3,2))")"; done
