python tools/e2e_timeline.py 2>&1 | grep ETD_TIMELINE > gpurun_out/r2_tl_shaped.txt
echo "$(grep -E ' (col[0-9]+|x0|down0|down[0-9]+) ' gpurun_out/r2_tl_shaped.txt | awk '{printf "%s=%s ", $2, $3}')"
timeout 600 python -m pytest tests/test_gpu_fold2.py tests/test_gpu_parity.py -q -x -k "pipelined" > gpurun_out/r2_tl_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2_tl_tests.log
timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu --no-alt --e2e-steps 3 > gpurun_out/r2_tl_bench.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/r2_tl_bench.json').read().strip().splitlines()[-1])
print(round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],1), 'pageable', round(d['e2e_pageable']['ms_per_step'],1))"
