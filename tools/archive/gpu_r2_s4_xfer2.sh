for v in "ETD_XFER_STREAMS=1" "ETD_XFER_STREAMS=2" "ETD_XFER_STREAMS=1" "ETD_XFER_STREAMS=2"; do
env $v python bench.py --steps 2 --warmup 3 --no-cpu --no-alt --no-e2e-pageable --e2e-steps 3 2> /dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['e2e']['ms_per_step'])"
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fold2.py tests/test_gpu_determinism.py -q -x 2>&1 | tail -2
