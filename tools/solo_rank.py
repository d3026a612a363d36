"""Per-rank compute time of the z-slab sharded schedule at G ranks, measured on ONE GPU
(dev tool): rank 0 of a G-rank plan runs its own ops -- pack, source, z stage on its
y-row chunks, y stack pass from the receive blocks, y and x stages, commit -- with the
exchanges skipped (ETD_SOLO_RANK; the peers' pieces read as zeros, so the VALUES are
meaningless; the launches, tiles and bytes are the real ones).  T(1) / (G x this time)
bounds the strong-scaling efficiency from the compute side: what sharding costs before
any byte crosses NVLink.  The exchanges themselves (NCCL) are not in this number.

python tools/solo_rank.py CFG G [G ...]      # e.g. 4 2 4 8"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["ETD_SOLO_RANK"] = "1"
import paper_2601_06849_b200 as etd  # noqa: E402
from paper_2601_06849_b200 import configs  # noqa: E402

cid = int(sys.argv[1])
cfg = configs.CONFIGS[cid]
n = int(os.environ.get("AB_N", cfg.n))
steps = 3
for G in [int(a) for a in sys.argv[2:]]:
    if G == 1:
        plan = configs.make_plan(cfg, n)
        for s, a in enumerate(configs.initial_state(cfg, n)):
            plan.upload(s, a)
        plan.step(1)
        t0 = time.perf_counter()
        plan.step(steps)                        # returns after the step's status readback
        ms = (time.perf_counter() - t0) / steps * 1e3
        rec = {"config": cid, "n": n, "G": 1, "ms_per_step": round(ms, 3)}
    else:
        plan = configs.make_plan(cfg, n, world_size=G, rank=0)
        z0, z1 = plan.slab
        for s in range(cfg.nspecies):
            plan.upload(s, etd.fill_config_ic(cfg.id, configs.SEED, s, n, z0, z1))
        etd.group_step([plan], 1)
        t0 = time.perf_counter()
        etd.group_step([plan], steps)          # synchronises the stream before returning
        ms = (time.perf_counter() - t0) / steps * 1e3
        rec = {"config": cid, "n": n, "G": G, "rank": 0, "slab_planes": z1 - z0, "ms_per_step_rank": round(ms, 3),
               "launches_per_step": plan.launches_per_step}
    plan.close()
    print(json.dumps(rec), flush=True)
