# A/B: fused backward tile classes (T=3: 2 CTAs/SM 2-stage; T=0: 1 CTA/SM 4-stage) on config 4
for X in 3 0; do for YZ in 3 0; do
ETD_BACK6_TILE_X=$X ETD_BACK6_TILE_YZ=$YZ timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --no-alt --no-e2e-pageable --e2e-steps 1 > gpurun_out/r2_tiles_${X}_${YZ}.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/r2_tiles_${X}_${YZ}.json').read().strip().splitlines()[-1])
st={s['name']:s['ms'] for s in d['roofline']['stages']}
print('X=$X YZ=$YZ', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],1), {k:v for k,v in st.items() if 'back' in k})"
done; done
