timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_fold2.py -q > gpurun_out/pytest_det.log 2>&1; echo "det tests rc=$?"; tail -4 gpurun_out/pytest_det.log
timeout 1200 python tools/tile_sweep.py 4 3 > gpurun_out/tile_sweep_l2.txt 2>&1; echo "sweep rc=$?"; cat gpurun_out/tile_sweep_l2.txt
