# session 4 final evidence: GPU suite, smoke, bench (+reference arm), launch list, ncu of the fused backward launches (config 3)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s4_pytest_gpu_final2.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/s4_pytest_gpu_final2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4_smoke_final2.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s4_smoke_final2.log
timeout 1200 python bench.py > gpurun_out/s4_bench_final2.json 2> gpurun_out/s4_bench_final2.err; echo "bench rc=$?"; tail -2 gpurun_out/s4_bench_final2.err
timeout 900 python bench.py --impl reference > gpurun_out/s4_bench_ref_final2.json 2> gpurun_out/s4_bench_ref_final2.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s4_launches_final2.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-alt --e2e-steps 1 --no-e2e-pageable > /dev/null 2>&1; echo "ncu list rc=$?"
M="--metrics sm__inst_executed_pipe_tensor_subpipe_dmma.sum"
timeout 900 ncu --set full $M --clock-control none -k regex:etd_back6 -c 10 -o gpurun_out/s4_fin_back6 python tools/one_step.py 3 > /dev/null 2>&1; echo "ncu back6 rc=$?"
python tools/ncu_summary.py gpurun_out/s4_fin_back6.ncu-rep z_back_a,z_back_b,z_back_c,z_back_d,y_back_a,y_back_b,y_back_c,y_back_d,x_back_src,x_back_upd gpurun_out/r02_ncu_full_cfg3_back6_s4.md > /dev/null 2>&1
rm -f gpurun_out/s4_fin_back6.ncu-rep
