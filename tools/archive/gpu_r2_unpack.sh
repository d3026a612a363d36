timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_fold2.py -q -x -k "sharded" > gpurun_out/r2_unpack_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2_unpack_tests.log
