# device setup bitwise check (small) + BASELINE configs[4] on one GPU
timeout 600 python tools/dsetup_check.py > gpurun_out/r2_dsetup2.log 2>&1; echo "check $?"; grep -c "bitwise: True" gpurun_out/r2_dsetup2.log; grep "MISMATCH\|bitwise: False" gpurun_out/r2_dsetup2.log
export AMGP_SETUP_TRACE=1
timeout 900 python bench.py --solve-only --gpus 1 --solve-scaling strong --weak-grid 512 --solve-stencil 27 --solve-k 3 --solve-family opt_cheb1 > gpurun_out/r2_s5_out1.log 2> gpurun_out/r2_s5_err1.log
echo "rc $?"; grep '^{' gpurun_out/r2_s5_out1.log; grep -v "amgp setup" gpurun_out/r2_s5_err1.log | tail -30
