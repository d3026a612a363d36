# round-2 session 4: verify the restored checkpoint (GPU suite, smoke, bench)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s4_pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/s4_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s4_smoke.log
timeout 1200 python bench.py --no-cpu > gpurun_out/s4_bench.json 2> gpurun_out/s4_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/s4_bench.err
