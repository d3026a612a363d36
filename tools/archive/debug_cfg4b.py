"""A/B the resident vs pipelined paths at full size (GPU only)."""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2601_06849_b200 as etd  # noqa: E402
from paper_2601_06849_b200 import configs  # noqa: E402
from oracle import rel_gap  # noqa: E402

n = int(sys.argv[1])
mode = sys.argv[2]
cfg = configs.CONFIGS[4]
path = f"/tmp/dbg_{n}_{mode}.npy"
if mode != "compare":
    u0, v0 = configs.initial_state(cfg, n)
    g = etd.unit_box_grid(3, n + 1)
    f = etd.fhn_cubic()
    plan = etd.make_system_plan(g, cfg.tau, 1e-3, 5e-4, 0.0, source=f)
    if mode.startswith("pipe"):
        st = etd.etd2rkds_step_system(plan, etd.SystemState(0, 0.0, u0, v0), f, nsteps=1)
        u = st.U
    else:
        plan.upload(0, u0)
        plan.upload(1, v0)
        if mode.startswith("prof"):
            plan.set_profiling(True)
        plan.step(1)
        u = plan.download(0)[0]
    np.save(path, u)
    sys.exit(0)
ref = np.load(f"/tmp/dbg_{n}_pipe.npy")
res = {}
for m in sys.argv[3:]:
    a = np.load(f"/tmp/dbg_{n}_{m}.npy")
    d = np.abs(a - ref).reshape(n, n, n)
    bad = np.where(d.max(axis=(1, 2)) > 1e-12)[0]
    badj = np.where(d.max(axis=(0, 2)) > 1e-12)[0]
    res[m] = {"gap": rel_gap(ref, a), "bad_planes": len(bad), "planes": bad[:12].tolist(),
              "bad_rows": len(badj), "rows": badj[:12].tolist()}
print(json.dumps(res))
