"""Config 4 full-length (20-step) parity against the reference CPU implementation,
split over two gpurun calls because one reference step takes ~190 s on the box's
host cores and a call is capped at one hour.

  python tools/parity_cfg4_full.py part1 OUT.jsonl   # reference steps 0 -> 10, ETRD checkpoint in /tmp
  python tools/parity_cfg4_full.py part2 OUT.jsonl   # restart from the checkpoint, steps 10 -> 20

Each part also runs the device path (default schedule, ETD_DENSE=1 dense
transforms, optionally ETD_BACK6=0: ETD_PARITY_SCHEDULES) to the same step and records max|a-b|/max|a| against the reference.
The checkpoint is written and read with the reference's own save_field /
load_field (ETRD, field.cpp:46-81), so the restart is the reference's own.  Part 2
needs part 1's checkpoint on the same box (gpurun reuses a box for a call that
starts within 5 minutes of the previous one; /tmp survives that).  Part 2 also
writes a strided sample of the reference state at step 20 (every 4099th point)
to gpurun_out/, a regression anchor for later schedules.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2601_06849_b200 as etd  # noqa: E402
from paper_2601_06849_b200 import configs  # noqa: E402
from oracle import Ref, rel_gap  # noqa: E402

CK = "/tmp/etd_cfg4_ref_step{step}_{sp}.etrd"
SAMPLE_STRIDE = 4099


SCHEDULES = {"default": {}, "dense": {"ETD_DENSE": "1"}, "r01_unfold": {"ETD_BACK6": "0"}}


def gpu_run(cfg, n, ics, steps, name):
    env = SCHEDULES[name]
    os.environ.update(env)
    try:
        plan = configs.make_plan(cfg, n)
    finally:
        for k in env:
            os.environ.pop(k, None)
    t0 = time.time()
    g = etd.etd2rkds_step_system(plan, etd.SystemState(0, 0.0, ics[0], ics[1]), cfg.source, nsteps=steps)
    sec = time.time() - t0
    lvl = plan.fold_level()
    plan.close()
    return [g.U, g.V], sec, lvl


def main():
    part, out = sys.argv[1], sys.argv[2]
    cfg = configs.CONFIGS[4]
    n = int(os.environ.get("ETD_PARITY_N", cfg.n))  # smaller n: dry runs of the script only
    cores = os.cpu_count() or 1
    Ref.set_threads(cores)
    s0, s1 = (0, 10) if part == "part1" else (10, 20)
    # reference first (it needs the most host memory), then the device runs one at a time
    if part == "part1":
        u, v = configs.initial_state(cfg, n)
    else:
        u, su, tu = Ref.load_field(CK.format(step=s0, sp="u"), n ** 3)
        v, sv, tv = Ref.load_field(CK.format(step=s0, sp="v"), n ** 3)
        assert abs(tu - s0 * cfg.tau) < 1e-12 and abs(tv - s0 * cfg.tau) < 1e-12, (tu, tv)
        u, v = np.ascontiguousarray(u), np.ascontiguousarray(v)
    t0 = time.time()
    r = Ref.system_run(cfg.dim, n, cfg.tau, cfg.kappa[0], cfg.kappa[1], cfg.q, u, v, s1 - s0, src_kind=10,
                       src_params=(0.1, 0.01, 0.5), n0=s0, t0=s0 * cfg.tau, lean=True, inplace=True)
    t_ref = time.time() - t0
    ref = [r[0], r[1]]
    del r
    if part == "part1":
        for a, sp in zip(ref, "uv"):
            Ref.save_field((n, n, n), a, s1 * cfg.tau, CK.format(step=s1, sp=sp))
    else:
        idx = np.arange(0, n ** 3, SAMPLE_STRIDE)
        np.savez(os.path.join(ROOT, "gpurun_out", "r02_cfg4_ref_step20_sample.npz"), idx=idx,
                 u=ref[0][idx], v=ref[1][idx], stride=SAMPLE_STRIDE)
    ics = configs.initial_state(cfg, n)
    # one record per schedule, written as soon as it is measured (a failing schedule
    # must not lose the reference run)
    for name in os.environ.get("ETD_PARITY_SCHEDULES", "default,dense").split(","):
        try:
            st, sec, lvl = gpu_run(cfg, n, ics, s1, name)
        except Exception as e:
            print(json.dumps({"schedule": name, "error": repr(e)}), flush=True)
            continue
        rec = {"config": 4, "n": n, "steps": s1, "reference_steps_this_call": [s0, s1],
               "schedule": name, "fold_level": list(lvl),
               "rel_gap": [rel_gap(a, b) for a, b in zip(ref, st)],
               "max_abs_diff": [float(np.max(np.abs(a - b))) for a, b in zip(ref, st)],
               "max_abs_ref": [float(np.max(np.abs(a))) for a in ref],
               "finite": [bool(np.all(np.isfinite(b))) for b in st],
               "tolerance": 1e-11, "gpu_wall_s": round(sec, 2), "ref_wall_s": round(t_ref, 1),
               "ref": (f"oracle/_ref (unmodified etdrd core, OpenBLAS {cores} threads), 3D two-species step "
                       "composed from reference primitives (system_stepper.cpp:74-114 + stepper.cpp:244-247)"
                       + ("" if part == "part1" else f"; restarted at step {s0} from the reference's own ETRD "
                                                       "save_field/load_field checkpoint"))}
        del st
        rec["pass"] = all(x <= 1e-11 for x in rec["rel_gap"]) and all(rec["finite"])
        print(json.dumps(rec), flush=True)
        with open(out, "a") as f:
            f.write(json.dumps(rec) + "\n")


if __name__ == "__main__":
    main()
