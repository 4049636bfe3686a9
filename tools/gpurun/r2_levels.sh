# schedule experiment for long-row levels: split vs deep thread-per-row
for v in 1 8 16 24; do AMGP_ROWS=$v timeout 300 python tools/level_bench.py --m 128 >> gpurun_out/r2_levels.jsonl 2>gpurun_out/r2_levels_err.log; echo "v$v $?"; done
for v in 1 16; do AMGP_ROWS=$v timeout 300 python tools/level_bench.py --m 256 --reps 20 >> gpurun_out/r2_levels.jsonl 2>>gpurun_out/r2_levels_err.log; echo "v$v 256 $?"; done
