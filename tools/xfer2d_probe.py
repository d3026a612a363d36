"""Pinned host->device rates of 2D strided copies by row width (dev tool): the
x-column-range upload of the pipelined advance copies (x1-x0)*8-byte pieces of
every (y, z) row."""
import ctypes as C
import time

import torch

rt = C.CDLL("/usr/local/cuda/lib64/libcudart.so")
nx, rows = 1024, 1024 * 1024            # 8 GB host field, 1023-wide rows padded to 1024
h = torch.empty(nx * rows, dtype=torch.float64).pin_memory()
d = torch.empty(nx * rows, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for width in (1024, 512, 256, 128, 64, 32):
    for kind, name in ((1, "H2D"), (2, "D2H")):
        best = 0.0
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for x0 in range(0, nx, width):
                dst, src = (d.data_ptr(), h.data_ptr()) if kind == 1 else (h.data_ptr(), d.data_ptr())
                rc = rt.cudaMemcpy2DAsync(C.c_void_p(dst + x0 * 8), C.c_size_t(nx * 8), C.c_void_p(src + x0 * 8),
                                          C.c_size_t(nx * 8), C.c_size_t(width * 8), C.c_size_t(rows), kind,
                                          C.c_void_p(0))
                assert rc == 0, rc
            torch.cuda.synchronize()
            best = max(best, nx * rows * 8 / (time.perf_counter() - t0) / 1e9)
        print(f"{name} row piece {width * 8:6d} B: {best:.1f} GB/s", flush=True)
