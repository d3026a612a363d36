"""A/B of environment switches on one config (dev tool): per-stage ms and a crc of
the state after the steps (bitwise comparison between variants).

python tools/ab_stage.py CFG STEPS STAGE_SUBSTR[,..] "" "ETD_X=1" "ETD_X=2 ETD_Y=0" ...
"""
import json
import os
import sys
import zlib

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06849_b200 import configs  # noqa: E402

cid, steps, subs = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3].split(",")
cfg = configs.CONFIGS[cid]
n = int(os.environ.get("AB_N", cfg.n))
ics = configs.initial_state(cfg, n)
for variant in sys.argv[4:]:
    env = dict(kv.split("=", 1) for kv in variant.split())
    os.environ.update(env)
    try:
        plan = configs.make_plan(cfg, n)
    finally:
        for k in env:
            os.environ.pop(k, None)
    for s, a in enumerate(ics):
        plan.upload(s, a)
    plan.step(1)
    plan.set_profiling(True)
    plan.step(steps)
    st = plan.stage_stats()
    plan.set_profiling(False)
    tot = sum(x["ms_total"] for x in st) / steps
    sel = {x["name"]: round(x["ms_total"] / max(1, x["launches"]), 3) for x in st
           if any(q in x["name"] for q in subs)}
    crc = zlib.crc32(plan.download(0)[0].tobytes())
    plan.close()
    print(json.dumps({"variant": variant or "default", "ms_per_step": round(tot, 2), "crc_u": crc, "stages": sel}),
          flush=True)
