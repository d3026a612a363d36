"""Per-stage device timing of the CUDA step on the BASELINE configs (dev tool).

python tools/quick_perf.py [cfg ids...] [--steps K] [--thomas]
Prints one JSON line per config with per-stage ms, TFLOP/s and pt-updates/s.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2601_06849_b200 import configs  # noqa: E402


def run(cfg_id: int, steps: int, n=None, **kw):
    cfg = configs.CONFIGS[cfg_id]
    n = cfg.n if n is None else n
    t0 = time.time()
    ics = configs.initial_state(cfg, n)
    t_ic = time.time() - t0
    plan = configs.make_plan(cfg, n, **kw)
    for s, a in enumerate(ics):
        plan.upload(s, a)
    plan.step(1)  # warm-up (graph build, L2)
    plan.set_profiling(True)
    plan.step(steps)
    st = plan.stage_stats()
    tot = sum(x["ms_total"] for x in st) / steps
    pts = cfg.points(n) * cfg.nspecies
    out = {"cfg": cfg_id, "backend": plan.backend.name, "n": n, "steps": steps, "ms_per_step": tot, "pt_upd_per_s": pts / (tot * 1e-3),
           "tflops": cfg.flops_per_step(n) / (tot * 1e-3) * 1e-12, "ic_s": round(t_ic, 2), "stages": []}
    for x in st:
        ms = x["ms_total"] / max(1, x["launches"])
        out["stages"].append({"name": x["name"], "ms": round(ms, 4),
                              "tflops": round(x["flops_per_launch"] / (ms * 1e-3) * 1e-12, 2),
                              "gbs": round(x["bytes_per_launch"] / (ms * 1e-3) * 1e-9, 1)})
    plan.set_profiling(False)
    # graph path timing
    import ctypes
    t1 = time.time()
    plan.step(steps)
    u, nn, tt = plan.download(0)
    out["graph_wall_ms_per_step"] = (time.time() - t1) / steps * 1e3
    out["finite"] = bool(np.all(np.isfinite(u)))
    plan.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    args = sys.argv[1:]
    steps = 3
    if "--steps" in args:
        i = args.index("--steps")
        steps = int(args[i + 1])
        del args[i:i + 2]
    kw = {}
    if "--thomas" in args:
        args.remove("--thomas")
        from paper_2601_06849_b200 import etd
        kw["backend"] = etd.BackendKind.Thomas
    ids = [int(a) for a in args] or [0, 1, 2, 3, 4]
    for c in ids:
        run(c, steps if c < 3 else min(steps, 2), **kw)
