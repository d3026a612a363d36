# fused source + level-2 stack: GPU tests, bench line, ncu of the dominant x_fwd_mix_odd launch
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu --no-alt > gpurun_out/bench_fs.json 2> gpurun_out/bench_fs.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_fs.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:etd_contract -s 7 -c 1 -o gpurun_out/xmix_odd_l2 python tools/one_step.py 4 > gpurun_out/ncu_full3.log 2>&1; echo "ncu full3 rc=$?"; tail -2 gpurun_out/ncu_full3.log
