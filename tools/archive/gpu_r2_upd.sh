timeout 900 python -m pytest tests/test_gpu_fold2.py tests/test_gpu_determinism.py tests/test_gpu_parity.py -q > gpurun_out/r2_upd_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2_upd_tests.log
timeout 300 python tools/check_cfg4_sample.py gpurun_out/r02_cfg4_sample_checks.jsonl back6_yz_transposed
timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu --no-alt --no-e2e-pageable --e2e-steps 2 > gpurun_out/r2_upd_bench.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/r2_upd_bench.json').read().strip().splitlines()[-1])
print(round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],1), {s['name']:s['ms'] for s in d['roofline']['stages'] if 'back' in s['name']})"
