# round-2 evidence run: full GPU suite, smoke, quick perf of configs 0-3, full-size parity of configs 0-3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_pytest_gpu_final.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2_pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke_final.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_smoke_final.log
timeout 600 python tools/quick_perf.py 0 1 2 3 > gpurun_out/r02_quick_perf_cfg0123.jsonl 2>&1; echo "quick rc=$?"
timeout 1800 python tools/parity_configs.py gpurun_out/r02_parity_configs_0123.jsonl 0 1 2 3 > gpurun_out/r2_parity0123.log 2>&1; echo "parity rc=$?"; tail -4 gpurun_out/r2_parity0123.log | cut -c1-200
