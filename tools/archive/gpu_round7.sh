timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -6 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu --no-alt > gpurun_out/bench7.json 2> gpurun_out/bench7.err; echo "bench rc=$?"; tail -2 gpurun_out/bench7.err
