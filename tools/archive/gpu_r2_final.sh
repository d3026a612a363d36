# round-2 final evidence: bench (+reference arm), launch list, ncu of the fused backward launches (config 3)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python bench.py > gpurun_out/r2_bench_final.json 2> gpurun_out/r2_bench_final.err; echo "bench rc=$?"; tail -2 gpurun_out/r2_bench_final.err
timeout 900 python bench.py --impl reference > gpurun_out/r2_bench_ref_final.json 2> gpurun_out/r2_bench_ref_final.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_final.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-alt --e2e-steps 1 --no-e2e-pageable > /dev/null 2>&1; echo "ncu list rc=$?"
M="--metrics sm__inst_executed_pipe_tensor_subpipe_dmma.sum"
timeout 900 ncu --set full $M --clock-control none -k regex:etd_back6 -c 6 -o gpurun_out/r2_fin_back6 python tools/one_step.py 3 > /dev/null 2>&1; echo "ncu back6 rc=$?"
python tools/ncu_summary.py gpurun_out/r2_fin_back6.ncu-rep z_back_a,z_back_b,y_back_a,y_back_b,x_back_src,x_back_upd gpurun_out/r02_ncu_full_cfg3_back6_final.md > /dev/null 2>&1
rm -f gpurun_out/r2_fin_back6.ncu-rep
