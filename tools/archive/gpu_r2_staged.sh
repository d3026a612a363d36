# staged x-stage epilogue of the fused backward: tests + config-4 sample parity + bench
timeout 900 python -m pytest tests/test_gpu_fold2.py tests/test_gpu_determinism.py -x -q > gpurun_out/r2_staged_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_staged_tests.log
timeout 300 python tools/check_cfg4_sample.py gpurun_out/r02_cfg4_sample_checks.jsonl back6_staged_x
timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu --no-alt --no-e2e-pageable > gpurun_out/r2_staged_bench.json 2> gpurun_out/r2_staged_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/r2_staged_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/r2_staged_bench.json').read().strip().splitlines()[-1])
print(round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],1), {s['name']:s['ms'] for s in d['roofline']['stages'] if 'x_' in s['name']})"
