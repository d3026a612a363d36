"""Host<->device transfer rates of the state upload/download path (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_06849_b200 import configs  # noqa: E402

cfg = configs.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
plan = configs.make_plan(cfg)
cnt = plan.local_count
h = torch.empty(cnt, dtype=torch.float64).pin_memory()
h.fill_(0.5)
for it in range(3):
    t0 = time.perf_counter()
    plan.upload_ptr(0, h.data_ptr(), cnt)
    t1 = time.perf_counter()
    plan.download_ptr(0, h.data_ptr(), cnt)
    t2 = time.perf_counter()
    print(f"upload {cnt*8/(t1-t0)/1e9:.1f} GB/s  download {cnt*8/(t2-t1)/1e9:.1f} GB/s")
d = torch.empty(cnt, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for it in range(2):
    t0 = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    h.copy_(d, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"contiguous torch H2D {cnt*8/(t1-t0)/1e9:.1f} GB/s  D2H {cnt*8/(t2-t1)/1e9:.1f} GB/s")
