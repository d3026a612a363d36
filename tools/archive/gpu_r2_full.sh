# round-2 evidence: full GPU suite, smoke, bench (+reference arm), launch list
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_pytest_gpu_full.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2_pytest_gpu_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_smoke.log
timeout 1200 python bench.py > gpurun_out/r2_bench_full.json 2> gpurun_out/r2_bench_full.err; echo "bench rc=$?"; tail -2 gpurun_out/r2_bench_full.err
timeout 900 python bench.py --impl reference > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-alt --e2e-steps 1 --no-e2e-pageable > gpurun_out/r2_ncu_launch.log 2>&1; echo "ncu list rc=$?"
