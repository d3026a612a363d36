# A/B: S=4 launches vs two S=2 launches (ETD_PAIRS=1) on every BASELINE config; GPU tests with both
timeout 900 python -m pytest tests/test_gpu_fold2.py tests/test_gpu_fold.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_a.log 2>&1; echo "tests default rc=$?"; tail -3 gpurun_out/pytest_a.log
ETD_PAIRS=1 timeout 900 python -m pytest tests/test_gpu_fold2.py tests/test_gpu_fold.py tests/test_gpu_sharded.py tests/test_gpu_determinism.py -q -x > gpurun_out/pytest_b.log 2>&1; echo "tests pairs rc=$?"; tail -3 gpurun_out/pytest_b.log
timeout 600 python tools/quick_perf.py 1 2 3 4 --steps 3 > gpurun_out/qp_default.jsonl 2>&1; echo "qp default rc=$?"
ETD_PAIRS=1 timeout 600 python tools/quick_perf.py 1 2 3 4 --steps 3 > gpurun_out/qp_pairs.jsonl 2>&1; echo "qp pairs rc=$?"
ETD_FOLD2=0 timeout 600 python tools/quick_perf.py 0 1 2 3 --steps 3 > gpurun_out/qp_l1.jsonl 2>&1; echo "qp l1 rc=$?"
timeout 300 python tools/quick_perf.py 0 --steps 20 > gpurun_out/qp_cfg0.jsonl 2>&1; echo "qp cfg0 rc=$?"
