# proxy-fenced consumer release: determinism + level-2 tests + config-4 sample parity + bench
timeout 120 python tools/back6_repeat.py 255 x_back_src,x_back_upd,z_back_a,y_back_a
timeout 120 python tools/back6_repeat.py 1023 x_back_src,x_back_upd
timeout 900 python -m pytest tests/test_gpu_fold2.py tests/test_gpu_determinism.py tests/test_gpu_sharded.py -x -q > gpurun_out/r2_fence_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_fence_tests.log
timeout 300 python tools/check_cfg4_sample.py gpurun_out/r02_cfg4_sample_checks.jsonl back6_fenced
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu --no-alt --no-e2e-pageable > gpurun_out/r2_fence_bench.json 2> gpurun_out/r2_fence_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/r2_fence_bench.err
