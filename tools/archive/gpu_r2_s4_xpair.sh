timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/s4_pytest_gpu5.log 2>&1; echo "gpu tests rc=$?"; tail -6 gpurun_out/s4_pytest_gpu5.log
