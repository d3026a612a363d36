"""Repeat-determinism of named stage kernels (etd_debug_repeat_op) at config-4
physics, n from argv; prints mismatching element counts and the (x, row) of the
first few."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2601_06849_b200 as etd  # noqa: E402
from paper_2601_06849_b200 import configs  # noqa: E402

n = int(sys.argv[1])
names = sys.argv[2].split(",")
cfg = configs.CONFIGS[4]
plan = configs.make_plan(cfg, n)
for s, a in enumerate(configs.initial_state(cfg, n)):
    plan.upload(s, a)
plan.step(1)
L = etd.lib()
L.etd_debug_repeat_op.argtypes = [C.c_void_p, C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_longlong), C.c_void_p, C.c_int]
pitch = (n + 31) // 32 * 32
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("ETD_"))
for name in names:
    for out in (0, 1):
        mm = C.c_longlong(-1)
        pos = (C.c_longlong * 8)()
        rc = L.etd_debug_repeat_op(plan.handle, name.encode(), out, 4, C.byref(mm), pos, 8)
        where = [(int(p % pitch), int(p // pitch)) for p in list(pos)[:min(8, max(0, mm.value))]]
        print(f"[{tag}] n={n} {name} out={out} rc={rc} mismatches={mm.value} (x,row)={where}", flush=True)
