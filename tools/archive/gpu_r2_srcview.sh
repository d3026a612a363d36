# per-SASS-instruction source view (bank conflicts, stalls) of x_fwd_mix_even_a and x_back_src, config 3
for spec in "x_fwd_mix_even_a:contract:8" "x_back_src:back6:4"; do
  name=${spec%%:*}; rest=${spec#*:}; kern=${rest%%:*}; skip=${rest##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:etd_$kern -s $skip -c 1 -o gpurun_out/r2_src_$name python tools/one_step.py 3 > /dev/null 2>&1; echo "$name rc=$?"
  ncu -i gpurun_out/r2_src_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_srcview_$name.csv 2>/dev/null
  rm -f gpurun_out/r2_src_$name.ncu-rep
  ls -la gpurun_out/r2_srcview_$name.csv
done
