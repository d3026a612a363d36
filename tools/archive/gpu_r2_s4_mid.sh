# session 4 mid-point evidence: GPU suite, bench, launch list, ncu of the new stack passes (config 3)
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s4_pytest_gpu3.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/s4_pytest_gpu3.log
timeout 1200 python bench.py --no-cpu > gpurun_out/s4_bench_mid.json 2> gpurun_out/s4_bench_mid.err; echo "bench rc=$?"; tail -2 gpurun_out/s4_bench_mid.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"etd_source|etd_fold2" -c 3 -o gpurun_out/s4_stack2 python tools/one_step.py 3 > /dev/null 2>&1; echo "ncu stack rc=$?"
