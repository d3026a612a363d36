"""Diagnose full-size (n=1023) 3D discrepancies: GPU resident vs pipelined paths,
and GPU vs the reference for (a) zero source (transforms only), (b) the config-4
FHN source, (c) a scalar 3D step.  One step each.  python tools/debug_cfg4.py [n]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2601_06849_b200 as etd  # noqa: E402
from paper_2601_06849_b200 import configs  # noqa: E402
from oracle import Ref, rel_gap  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1023
Ref.set_threads(os.cpu_count())
cfg = configs.CONFIGS[4]
u0, v0 = configs.initial_state(cfg, n)
g = etd.unit_box_grid(3, n + 1)
out = {"n": n}


def gpu_system(src, pipelined):
    plan = etd.make_system_plan(g, cfg.tau, 1e-3, 5e-4, 0.0, source=src)
    if pipelined:
        st = etd.etd2rkds_step_system(plan, etd.SystemState(0, 0.0, u0, v0), src, nsteps=1)
        r = (st.U, st.V)
    else:
        plan.upload(0, u0)
        plan.upload(1, v0)
        plan.step(1)
        r = (plan.download(0)[0], plan.download(1)[0])
    plan.close()
    return r


a = gpu_system(etd.fhn_cubic(), False)
b = gpu_system(etd.fhn_cubic(), True)
out["resident_vs_pipelined_bitwise"] = [bool(np.array_equal(a[0], b[0])), bool(np.array_equal(a[1], b[1]))]
out["resident_vs_pipelined_gap"] = [rel_gap(a[0], b[0]), rel_gap(a[1], b[1])]
print(json.dumps(out), flush=True)
t0 = time.time()
r = Ref.system_run(3, n, cfg.tau, 1e-3, 5e-4, 0.0, u0, v0, 1, src_kind=10, src_params=(0.1, 0.01, 0.5), lean=True)
out["fhn_gap_resident"] = [rel_gap(r[0], a[0]), rel_gap(r[1], a[1])]
diff = np.abs(r[0] - a[0]).reshape(n, n, n)
kz, jy, ix = np.unravel_index(np.argmax(diff), diff.shape)
out["fhn_worst_u_at_kji"] = [int(kz), int(jy), int(ix)]
out["fhn_u_bad_planes"] = int(np.sum(diff.max(axis=(1, 2)) > 1e-12))
out["fhn_u_bad_rows_j"] = int(np.sum(diff.max(axis=(0, 2)) > 1e-12))
out["fhn_u_bad_cols_i"] = int(np.sum(diff.max(axis=(0, 1)) > 1e-12))
out["ref_s"] = round(time.time() - t0, 1)
print(json.dumps(out), flush=True)
z = gpu_system(etd.DeviceSource(etd.SourceKind.ZERO), False)
r = Ref.system_run(3, n, cfg.tau, 1e-3, 5e-4, 0.0, u0, v0, 1, src_kind=0, lean=True)
out["zero_src_gap"] = [rel_gap(r[0], z[0]), rel_gap(r[1], z[1])]
print(json.dumps(out), flush=True)
plan = etd.make_plan(g, 1e-3, 0.1, 1.0)
s = etd.advance(plan, etd.StepperState(0, 0.0, u0), etd.allen_cahn_cubic(), nsteps=1).U
plan.close()
r = Ref.scalar_run(3, n, 1e-3, 0.1, 1.0, u0, 1, src_kind=1)[0]
out["scalar_ac_gap"] = rel_gap(r, s)
print(json.dumps(out), flush=True)
