# user-spectra + smooth parity (one gpurun call), then the full GPU suite
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "user or spectra_check" > gpurun_out/pytest_user.log 2>&1; echo "pytest user exit $?"; tail -30 gpurun_out/pytest_user.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest all exit $?"; tail -5 gpurun_out/pytest_gpu.log
