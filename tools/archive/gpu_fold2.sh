# level-2 split validation: GPU tests, then the config-4 bench line
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests/test_gpu_fold2.py -x -q > gpurun_out/pytest_fold2.log 2>&1; echo "fold2 tests rc=$?"; tail -30 gpurun_out/pytest_fold2.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu --no-alt > gpurun_out/bench_l2.json 2> gpurun_out/bench_l2.err; echo "bench l2 rc=$?"; tail -3 gpurun_out/bench_l2.err
