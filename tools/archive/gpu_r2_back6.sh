# fused level-2 backward (etd_back6): GPU tests of the level-2 path + a config-4 bench line
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 600 python -m pytest tests/test_gpu_fold2.py tests/test_gpu_sharded.py -x -q > gpurun_out/r2_back6_tests.log 2>&1; echo "fold2 tests rc=$?"; tail -3 gpurun_out/r2_back6_tests.log
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "default_level2 or pipelined or system_steps" > gpurun_out/r2_back6_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/r2_back6_parity.log
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu --no-alt --no-e2e-pageable > gpurun_out/r2_back6_bench.json 2> gpurun_out/r2_back6_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/r2_back6_bench.err
