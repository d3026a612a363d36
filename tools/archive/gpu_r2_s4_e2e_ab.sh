for v in "ETD_SRC_L2=0 ETD_FOLDX4=0" "ETD_SRC_L2=3 ETD_FOLDX4=1" "ETD_SRC_L2=0 ETD_FOLDX4=1" "ETD_SRC_L2=3 ETD_FOLDX4=0"; do
env $v python bench.py --steps 2 --warmup 3 --no-cpu --no-alt --no-e2e-pageable --e2e-steps 3 2> /dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['e2e']['ms_per_step'])"
done
