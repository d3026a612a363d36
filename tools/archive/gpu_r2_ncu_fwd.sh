# ncu: z_fwd_even_a (MODE 1 forward, 0.87) vs x_fwd_mix_even_a (MODE 0 forward, 0.93), config 3
for spec in "z_fwd_even_a:0" "x_fwd_mix_even_a:8" "z_back_a:-"; do
  name=${spec%%:*}; skip=${spec##*:}
  if [ "$skip" = "-" ]; then K="regex:etd_back6"; S=0; else K="regex:etd_contract"; S=$skip; fi
  timeout 600 ncu --set full --clock-control none --import-source on -k $K -s $S -c 1 -o gpurun_out/r2_$name python tools/one_step.py 3 > gpurun_out/r2_ncu_$name.log 2>&1; echo "$name rc=$?"
  python tools/ncu_summary.py gpurun_out/r2_$name.ncu-rep $name gpurun_out/r2_ncu_cfg3_$name.md > /dev/null 2>&1
  python tools/ncu_hotspots.py gpurun_out/r2_$name.ncu-rep gpurun_out/r2_hotspots_$name.txt > /dev/null 2>&1
  ncu -i gpurun_out/r2_$name.ncu-rep --page details --csv > gpurun_out/r2_details_$name.csv 2>/dev/null
  ncu -i gpurun_out/r2_$name.ncu-rep --page raw --csv > gpurun_out/r2_raw_$name.csv 2>/dev/null
  rm -f gpurun_out/r2_$name.ncu-rep
done
