timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s4_pytest_gpu4.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/s4_pytest_gpu4.log
python tools/quick_perf.py 4 --steps 2 --thomas 2> /dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], [(s['name'], s['ms'], s['gbs']) for s in d['stages']])"
ETD_DENSE=1 python tools/ab_stage.py 3 2 source "" 2>/dev/null | cut -c1-200
