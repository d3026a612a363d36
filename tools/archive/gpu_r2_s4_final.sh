# session 4 evidence: GPU suite (incl. the full-size anchors), smoke, bench (+reference arm), launch list
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s4_pytest_gpu_final.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/s4_pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4_smoke_final.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s4_smoke_final.log
timeout 1200 python bench.py > gpurun_out/s4_bench_final.json 2> gpurun_out/s4_bench_final.err; echo "bench rc=$?"; tail -2 gpurun_out/s4_bench_final.err
timeout 900 python bench.py --impl reference > gpurun_out/s4_bench_ref_final.json 2> gpurun_out/s4_bench_ref_final.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4_launches_final.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-alt --e2e-steps 1 --no-e2e-pageable > /dev/null 2>&1; echo "ncu list rc=$?"
