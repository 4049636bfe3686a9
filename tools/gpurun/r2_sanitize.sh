# compute-sanitizer, one tool per call: bash tools/gpurun/r2_sanitize.sh <tool>
t=$1
timeout 300 python tools/sanitize_smoke.py > gpurun_out/r2_san_plain_$t.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 2400 compute-sanitizer --tool $t --error-exitcode 9 --print-limit 50 python tools/sanitize_smoke.py > gpurun_out/r2_sanitize_$t.log 2>&1
echo "sanitizer $t rc $?"
