"""Timeline of one pipelined host-buffer advance (ETD_TIMELINE): when each upload
chunk lands, each column chunk's z/y stages finish, each x-stage row chunk finishes
and each download chunk lands (ms from the call's start, device clock)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2601_06849_b200 import configs  # noqa: E402

cfg = configs.CONFIGS[4]
n = int(sys.argv[1]) if len(sys.argv) > 1 else cfg.n
ics = configs.initial_state(cfg, n)
plan = configs.make_plan(cfg, n)
pageable = len(sys.argv) > 2 and sys.argv[2] == "pageable"
if pageable:  # plain numpy (the reference Field's storage): staged through the plan's pinned mirror
    hin = [torch.from_numpy(a) for a in ics]
    hout = [torch.empty_like(h) for h in hin]
else:
    hin = [torch.from_numpy(a).pin_memory() for a in ics]
    hout = [torch.empty_like(h).pin_memory() for h in hin]
import time  # noqa: E402
for rep in range(2):
    if rep == 1:
        os.environ["ETD_TIMELINE"] = "1"
        if pageable:
            hout = [torch.empty_like(h) for h in hin]  # fresh pages, as a new Field per call
    t0 = time.perf_counter()
    r = plan.advance_ptr(hin[0].data_ptr(), hin[1].data_ptr(), hout[0].data_ptr(), hout[1].data_ptr(), 0, 0.0, 1)
    print("call", rep, r, "wall ms", round((time.perf_counter() - t0) * 1e3, 1), flush=True)
