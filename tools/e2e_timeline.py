"""Event timeline of the pipelined host-buffer advance (etd_advance) on a BASELINE
config: ETD_TIMELINE=1 python tools/e2e_timeline.py [CFG]  (dev tool; prints the
upload / column-stage / x-stage chunk events in ms from the call's start)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_06849_b200 import configs  # noqa: E402

cfg = configs.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
n = cfg.n
ics = configs.initial_state(cfg, n)
plan = configs.make_plan(cfg, n)
hin = [torch.from_numpy(a).pin_memory() for a in ics]
hout = [torch.empty_like(h).pin_memory() for h in hin]
ptr = lambda lst, i: lst[i].data_ptr() if i < len(lst) else 0
for it in range(2):
    print(f"--- call {it}", file=sys.stderr, flush=True)
    plan.advance_ptr(ptr(hin, 0), ptr(hin, 1), ptr(hout, 0), ptr(hout, 1), 0, 0.0, 1)
