"""Diagnostics for the fused level-2 backward (etd_back6): kernel determinism via
etd_debug_repeat_op, and where the pipelined host-buffer advance differs from the
device-resident steps (first differing (x, y, z), per species)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2601_06849_b200 as etd  # noqa: E402
from paper_2601_06849_b200 import configs  # noqa: E402

cfg = configs.CONFIGS[4]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 255
ics = configs.initial_state(cfg, n)
plan = configs.make_plan(cfg, n)
print("fold", plan.fold_level(), "stages", [s["name"] for s in plan.stage_stats()])
for s, a in enumerate(ics):
    plan.upload(s, a)
plan.step(1)
L = etd.lib()
L.etd_debug_repeat_op.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_longlong), C.c_void_p, C.c_int]
for st in plan.stage_stats():
    if st["flops_per_launch"] <= 0:
        continue
    for out in (0, 1):
        mm = C.c_longlong(-1)
        pos = (C.c_longlong * 4)()
        rc = L.etd_debug_repeat_op(plan.handle, st["name"].encode(), out, 4, C.byref(mm), pos, 4)
        print("repeat", st["name"], out, rc, mm.value, list(pos) if mm.value else "")
plan.close()
for chunks in ("1", "16"):
    for steps in (1, 2):
        os.environ["ETD_XFER_CHUNKS"] = chunks
        p = configs.make_plan(cfg, n)
        a = etd.etd2rkds_step_system(p, etd.SystemState(0, 0.0, *ics), cfg.source, nsteps=steps)
        for s, x in enumerate(ics):
            p.upload(s, x)
        p.step(steps)
        for s, got in enumerate((a.U, a.V)):
            ref = p.download(s)[0]
            d = np.nonzero(got != ref)[0]
            where = [(int(i % n), int(i // n % n), int(i // (n * n))) for i in d[:5]]
            print(f"chunks={chunks} steps={steps} species={s} ndiff={d.size} maxabs={np.max(np.abs(got-ref)):.3e} first={where}")
        p.close()
