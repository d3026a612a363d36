"""Full-size gap between the parity-split and the dense transform paths on a
BASELINE config (GPU only; the dense path's own gap to the reference CPU
implementation is in profiles/r01_parity_configs.jsonl).

python tools/fold_vs_dense.py OUT.jsonl CFG[:STEPS] ...
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2601_06849_b200 import configs  # noqa: E402
from oracle import rel_gap  # noqa: E402


def run(cfg, n, steps, ics, dense):
    if dense:
        os.environ["ETD_DENSE"] = "1"
    try:
        plan = configs.make_plan(cfg, n)
    finally:
        os.environ.pop("ETD_DENSE", None)
    split = plan.parity_split()
    for s, a in enumerate(ics):
        plan.upload(s, a)
    t0 = time.time()
    plan.step(steps)
    out = [plan.download(s)[0] for s in range(len(ics))]
    dt = time.time() - t0
    plan.close()
    return out, split, dt


def main():
    dst = sys.argv[1]
    for spec in sys.argv[2:]:
        cid = int(spec.split(":")[0])
        cfg = configs.CONFIGS[cid]
        steps = int(spec.split(":")[1]) if ":" in spec else cfg.steps
        ics = configs.initial_state(cfg, cfg.n)
        f, split, tf = run(cfg, cfg.n, steps, ics, False)
        d, _, td = run(cfg, cfg.n, steps, ics, True)
        rec = {"config": cid, "n": cfg.n, "steps": steps, "parity_split": list(split),
               "rel_gap_fold_vs_dense": [rel_gap(b, a) for a, b in zip(f, d)],
               "finite": [bool(np.all(np.isfinite(a))) for a in f], "fold_s": round(tf, 2), "dense_s": round(td, 2)}
        print(json.dumps(rec), flush=True)
        with open(dst, "a") as fh:
            fh.write(json.dumps(rec) + "\n")


if __name__ == "__main__":
    main()
