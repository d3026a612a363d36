#!/bin/bash
# A/B of prebuilt library variants: per-stage Thomas times on configs 3 and 4
for v in half updg; do
  cp tools/_variants/libetd_$v.so paper_2601_06849_b200/libetd_b200.so
  echo "== $v"
  python tools/quick_perf.py 3 4 --thomas 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print(d['cfg'], round(d['ms_per_step'], 2), ' '.join(f\"{s['name']}={s['ms']:.2f}\" for s in d['stages']))
"
done
cp tools/_variants/libetd_updg.so paper_2601_06849_b200/libetd_b200.so
timeout 900 python -m pytest tests/test_gpu_thomas.py tests/test_gpu_gate5.py tests/test_gpu_sharded.py tests/test_gpu_paper_tables.py -q -x 2>&1 | tail -3
