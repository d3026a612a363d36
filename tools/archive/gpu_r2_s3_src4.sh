# per-SASS source view + raw metrics of four config-4 launches (z_fwd_even_a, z_back_a, x_fwd_mix_even_a, x_back_src)
for spec in "z_fwd_even_a:contract:0" "z_back_a:back6:0" "x_fwd_mix_even_a:contract:8" "x_back_src:back6:4"; do
  name=${spec%%:*}; rest=${spec#*:}; kern=${rest%%:*}; skip=${rest##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:etd_$kern -s $skip -c 1 -o gpurun_out/s3_src4_$name python tools/one_step.py 4 > gpurun_out/s3_src4_$name.log 2>&1; echo "$name rc=$?"
  ncu -i gpurun_out/s3_src4_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/s3_src4_$name.csv 2>/dev/null
  ncu -i gpurun_out/s3_src4_$name.ncu-rep --page raw --csv > gpurun_out/s3_raw4_$name.csv 2>/dev/null
  rm -f gpurun_out/s3_src4_$name.ncu-rep
done
ls -la gpurun_out
