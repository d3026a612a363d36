# defaults: size-thresholded level 2 + pair launches: GPU tests, smoke, full bench, reference, launch list, ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -8 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/bench.err
timeout 600 python tools/quick_perf.py 0 1 2 3 --steps 5 > gpurun_out/qp_all.jsonl 2>&1; echo "qp rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-alt --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:etd_contract -s 19 -c 1 -o gpurun_out/xmix_odd_b python tools/one_step.py 4 > gpurun_out/ncu_full4.log 2>&1; echo "ncu full4 rc=$?"; tail -2 gpurun_out/ncu_full4.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:etd_unfold2 -s 2 -c 1 -o gpurun_out/unfold_src python tools/one_step.py 4 > gpurun_out/ncu_full5.log 2>&1; echo "ncu full5 rc=$?"; tail -2 gpurun_out/ncu_full5.log
