"""Pinned host <-> device copy rates for config 4's per-step bytes (2 fields of
1023^3 doubles each way), to put the e2e step time next to the PCIe floor (dev tool)."""
import time

import torch

n = 1023 ** 3
h = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(2)]
d = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(2):
        d[i].copy_(h[i], non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for i in range(2):
        h[i].copy_(d[i], non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    s = torch.cuda.Stream()
    t3 = time.perf_counter()
    for i in range(2):
        d[i].copy_(h[i], non_blocking=True)
    with torch.cuda.stream(s):
        for i in range(2):
            h[i].copy_(d[i], non_blocking=True)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
gb = 2 * n * 8 / 1e9
print(f"H2D {gb:.2f} GB in {(t1-t0)*1e3:.1f} ms ({gb/(t1-t0):.1f} GB/s); D2H {(t2-t1)*1e3:.1f} ms ({gb/(t2-t1):.1f} GB/s); "
      f"both directions concurrently {(t4-t3)*1e3:.1f} ms")
