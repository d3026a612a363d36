"""Re-run one stage kernel on unchanged inputs and locate nondeterministic outputs."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2601_06849_b200 as etd  # noqa: E402
from paper_2601_06849_b200 import configs  # noqa: E402

n = int(sys.argv[1])
names = sys.argv[2:] or ["x_fwd_corr"]
cfg = configs.CONFIGS[4]
u0, v0 = configs.initial_state(cfg, n)
g = etd.unit_box_grid(3, n + 1)
plan = etd.make_system_plan(g, cfg.tau, 1e-3, 5e-4, 0.0, source=etd.fhn_cubic())
plan.upload(0, u0)
plan.upload(1, v0)
plan.step(1)
L = etd.lib()
L.etd_debug_repeat_op.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_longlong),
                                  C.c_void_p, C.c_int]
pitch = (n + 31) // 32 * 32
for name in names:
    for out in (0, 1):
        mm = C.c_longlong()
        pos = np.zeros(64, dtype=np.int64)
        rc = L.etd_debug_repeat_op(plan.handle, name.encode(), out, 4, C.byref(mm), pos.ctypes.data_as(C.c_void_p), 64)
        k = min(64, mm.value)
        p = np.sort(pos[:k])
        rows, cols = p // pitch, p % pitch
        print(json.dumps({"op": name, "out": out, "rc": rc, "mismatches": mm.value,
                          "rows": rows[:16].tolist(), "cols": cols[:16].tolist(),
                          "rows_mod64": sorted(set((rows % 64).tolist()))[:16]}), flush=True)
