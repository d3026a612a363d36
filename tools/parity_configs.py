"""Full-size parity of the CUDA path against the reference CPU implementation on
all five BASELINE configs (north_star: max|a-b|/max|a| <= 1e-11 after the stated
number of steps).  Runs on the GPU box: the GPU result first, then the reference
(oracle/_ref: the unmodified etdrd core + OpenBLAS on all host cores) on the
same seeded inputs.  Appends one JSON line per config to the output file.

python tools/parity_configs.py OUT.jsonl [cfg ids]   (default 0 1 2 3 4; "4:2" = config 4, 2 steps)
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


def main():
    out = sys.argv[1]
    ids = sys.argv[2:] or ["0", "1", "2", "3", "4"]
    cores = os.cpu_count() or 1
    Ref.set_threads(cores)
    for spec in ids:
        cid = int(spec.split(":")[0])
        cfg = configs.CONFIGS[cid]
        n, steps = cfg.n, (int(spec.split(":")[1]) if ":" in spec else cfg.steps)
        ics = configs.initial_state(cfg, n)
        plan = configs.make_plan(cfg, n)
        t0 = time.time()
        if cfg.nspecies == 1:
            g = etd.advance(plan, etd.StepperState(0, 0.0, ics[0]), cfg.source, nsteps=steps)
            gpu = [g.U]
        else:
            g = etd.etd2rkds_step_system(plan, etd.SystemState(0, 0.0, ics[0], ics[1]), cfg.source, nsteps=steps)
            gpu = [g.U, g.V]
        t_gpu = time.time() - t0
        plan.close()
        del g
        t0 = time.time()
        if cfg.nspecies == 1:
            ref = [Ref.scalar_run(cfg.dim, n, cfg.tau, cfg.kappa[0], cfg.q, ics[0], steps, src_kind=1)[0]]
        else:
            r = Ref.system_run(cfg.dim, n, cfg.tau, cfg.kappa[0], cfg.kappa[1], cfg.q, ics[0], ics[1], steps,
                               src_kind=10, src_params=(0.1, 0.01, 0.5), lean=True, inplace=True)
            ref = [r[0], r[1]]
        t_ref = time.time() - t0
        rec = {"config": cid, "dim": cfg.dim, "n": n, "steps": steps, "config_steps": cfg.steps,
               "species": cfg.nspecies,
               "rel_gap": [rel_gap(a, b) for a, b in zip(ref, gpu)],
               "max_abs_diff": [float(np.max(np.abs(a - b))) for a, b in zip(ref, gpu)],
               "max_abs_ref": [float(np.max(np.abs(a))) for a in ref],
               "finite": [bool(np.all(np.isfinite(b))) for b in gpu],
               "tolerance": 1e-11, "gpu_wall_s": round(t_gpu, 2), "ref_wall_s": round(t_ref, 1),
               "ref": f"oracle/_ref (unmodified etdrd core, OpenBLAS {cores} threads)"
                      + ("" if cfg.nspecies == 1 else ", 3D two-species step composed from reference primitives")}
        rec["pass"] = all(x <= 1e-11 for x in rec["rel_gap"]) and all(rec["finite"])
        print(json.dumps(rec), flush=True)
        with open(out, "a") as f:
            f.write(json.dumps(rec) + "\n")
        del ics, gpu, ref


if __name__ == "__main__":
    main()
