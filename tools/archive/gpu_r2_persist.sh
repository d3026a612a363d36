# persistent etd_contract: determinism, level-2 tests, bench A/B (ETD_PERSIST=0/1)
timeout 900 python -m pytest tests/test_gpu_fold2.py tests/test_gpu_determinism.py tests/test_gpu_fold.py -x -q > gpurun_out/r2_persist_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2_persist_tests.log
for P in 1 0; do
ETD_PERSIST=$P timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu --no-alt --no-e2e-pageable --e2e-steps 1 > gpurun_out/r2_persist_$P.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/r2_persist_$P.json').read().strip().splitlines()[-1])
st={s['name']:(s['ms'],s['frac']) for s in d['roofline']['stages'] if s['bound']=='tensor' and ('_a' in s['name'] or 'corr' in s['name'])}
print('PERSIST=$P', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],1), st)"
done
timeout 300 python tools/check_cfg4_sample.py gpurun_out/r02_cfg4_sample_checks.jsonl persistent_contract
