timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -8 gpurun_out/pytest_gpu.log
timeout 600 python tools/quick_perf.py 1 2 3 4 --steps 3 > gpurun_out/qp6.jsonl 2>&1; echo "qp rc=$?"
timeout 900 python tools/fold_vs_dense.py gpurun_out/l2_vs_dense6.jsonl 1 2 3 4 > gpurun_out/l2_vs_dense6.log 2>&1; echo "vs dense rc=$?"; cut -c1-250 gpurun_out/l2_vs_dense6.jsonl
timeout 600 python tools/parity_configs.py gpurun_out/parity6.jsonl 0 1 2 > gpurun_out/parity6.log 2>&1; echo "parity rc=$?"; cut -c1-200 gpurun_out/parity6.jsonl
