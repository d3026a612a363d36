for D in 0 1; do
if [ $D = 1 ]; then export ETD_DBG_NOD=1; fi
timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu --no-alt --no-e2e-pageable --e2e-steps 1 > gpurun_out/r2_nod_$D.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/r2_nod_$D.json').read().strip().splitlines()[-1])
st={s['name']:(s['ms'],s['frac']) for s in d['roofline']['stages'] if s['bound']=='tensor' and ('_a' in s['name'] or 'corr' in s['name'])}
print('NOD=$D', round(d['ms_per_step'],2), st); print(json.dumps({k:d['roofline'][k] for k in ('kernel','achieved','frac','traffic','traffic_stage','kernel_share_of_step','slowest_launch')}))"
done
