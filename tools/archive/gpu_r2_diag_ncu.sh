# back6 diagnostics (determinism, pipelined vs resident) + ncu of the config-3 back6 / contract launches
timeout 600 python tools/back6_diag.py 255 > gpurun_out/r2_back6_diag.log 2>&1; echo "diag rc=$?"; tail -30 gpurun_out/r2_back6_diag.log
M="--metrics sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum"
timeout 900 ncu --set full $M --clock-control none --import-source on -k regex:etd_back6 -c 6 -o gpurun_out/r2_cfg3_back6 python tools/one_step.py 3 > gpurun_out/r2_ncu_back6.log 2>&1; echo "ncu back6 rc=$?"; tail -2 gpurun_out/r2_ncu_back6.log
python tools/ncu_summary.py gpurun_out/r2_cfg3_back6.ncu-rep z_back_a,z_back_b,y_back_a,y_back_b,x_back_src,x_back_upd gpurun_out/r2_ncu_cfg3_back6.md > /dev/null 2>&1
python tools/ncu_hotspots.py gpurun_out/r2_cfg3_back6.ncu-rep gpurun_out/r2_hotspots_cfg3_zback6.txt > /dev/null 2>&1
timeout 900 ncu --set full $M --clock-control none --import-source on -k regex:etd_contract -c 14 -o gpurun_out/r2_cfg3_contract python tools/one_step.py 3 > gpurun_out/r2_ncu_contract.log 2>&1; echo "ncu contract rc=$?"
python tools/ncu_summary.py gpurun_out/r2_cfg3_contract.ncu-rep z_fwd_even_a,z_fwd_even_b,z_fwd_odd_a,z_fwd_odd_b,y_fwd_even_a,y_fwd_even_b,y_fwd_odd_a,y_fwd_odd_b,x_fwd_mix_even_a,x_fwd_mix_even_b,x_fwd_mix_odd_a,x_fwd_mix_odd_b,x_fwd_corr_even,x_fwd_corr_odd gpurun_out/r2_ncu_cfg3_contract.md > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
for f in gpurun_out/*.ncu-rep; do s=$(stat -c %s $f); if [ $s -gt 25000000 ]; then echo "dropping $f ($s)"; rm $f; fi; done
