# 4 GPUs: whole gpu suite with the reference staged, smoke
R=$GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/r2_full_pytest.log 2>&1; echo "pytest $?"; tail -4 gpurun_out/r2_full_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_full_smoke.log 2>&1; echo "smoke $?"; tail -1 gpurun_out/r2_full_smoke.log
