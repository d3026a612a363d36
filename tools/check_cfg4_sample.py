"""Config 4 after its 20 steps on the device (default schedule, or the ETD_* switches
in the environment) against the reference CPU implementation's state at step 20,
sampled at every 4099th point (profiles/r02_cfg4_ref_step20_sample.npz, written by
tools/parity_cfg4_full.py part 2 from the full reference run).  The gap is
max|a-b| over the sample / max|ref| of the FULL reference field (from
profiles/r02_parity_cfg4_full.jsonl), the north star's normwise metric restricted
to the sampled points.

python tools/check_cfg4_sample.py OUT.jsonl [label]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2601_06849_b200 as etd  # noqa: E402
from paper_2601_06849_b200 import configs  # noqa: E402

out = sys.argv[1]
label = sys.argv[2] if len(sys.argv) > 2 else "default"
z = np.load(os.path.join(ROOT, "profiles", "r02_cfg4_ref_step20_sample.npz"))
stride = int(z["stride"])
ref_max = None
for line in open(os.path.join(ROOT, "profiles", "r02_parity_cfg4_full.jsonl")):
    r = json.loads(line)
    if r.get("steps") == 20 and "max_abs_ref" in r:
        ref_max = r["max_abs_ref"]
cfg = configs.CONFIGS[4]
n = cfg.n
ics = configs.initial_state(cfg, n)
plan = configs.make_plan(cfg, n)
for s, a in enumerate(ics):
    plan.upload(s, a)
t0 = time.time()
plan.step(cfg.steps)
sec = time.time() - t0
idx = np.arange(0, n ** 3, stride)
rec = {"config": 4, "steps": cfg.steps, "schedule": label, "fold_level": list(plan.fold_level()),
       "sample_stride": stride, "sample_points": int(idx.size)}
gaps = []
for s, key in enumerate("uv"):
    got = plan.download(s)[0][idx]
    d = float(np.max(np.abs(got - z[key])))
    gaps.append(d / ref_max[s])
rec.update({"rel_gap_sampled": gaps, "tolerance": 1e-11, "pass": all(g <= 1e-11 for g in gaps),
            "device_s": round(sec, 2)})
print(json.dumps(rec), flush=True)
with open(out, "a") as f:
    f.write(json.dumps(rec) + "\n")
