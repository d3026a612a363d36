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
hin = [torch.from_numpy(a).pin_memory() for a in ics]
hout = [torch.empty_like(h).pin_memory() for h in hin]
for rep in range(2):
    if rep == 1:
        os.environ["ETD_TIMELINE"] = "1"
    r = plan.advance_ptr(hin[0].data_ptr(), hin[1].data_ptr(), hout[0].data_ptr(), hout[1].data_ptr(), 0, 0.0, 1)
    print("call", rep, r, flush=True)
