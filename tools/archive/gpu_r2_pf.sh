# L2 prefetch of the x-stage aux tile in etd_back6: bench + ncu of x_back_src (config 3)
timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu --no-alt --no-e2e-pageable --e2e-steps 1 > gpurun_out/r2_pf_bench.json 2>/dev/null; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/r2_pf_bench.json').read().strip().splitlines()[-1])
print(round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],1), {s['name']:s['ms'] for s in d['roofline']['stages'] if 'back' in s['name']})"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:etd_back6 -s 4 -c 2 -o gpurun_out/r2_xsrc python tools/one_step.py 3 > gpurun_out/r2_ncu_xsrc.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py gpurun_out/r2_xsrc.ncu-rep x_back_src,x_back_upd gpurun_out/r2_ncu_cfg3_xsrc.md > /dev/null 2>&1; cat gpurun_out/r2_ncu_cfg3_xsrc.md
python tools/ncu_hotspots.py gpurun_out/r2_xsrc.ncu-rep gpurun_out/r2_hotspots_xsrc.txt > /dev/null 2>&1; head -30 gpurun_out/r2_hotspots_xsrc.txt
ncu -i gpurun_out/r2_xsrc.ncu-rep --page details --csv > gpurun_out/r2_xsrc_details.csv 2>/dev/null
rm -f gpurun_out/r2_xsrc.ncu-rep
