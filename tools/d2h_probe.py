import ctypes as C, time, torch
rt = C.CDLL("/usr/local/cuda/lib64/libcudart.so")
nx, rows = 1023, 1023*1023
h = torch.empty(nx*rows, dtype=torch.float64).pin_memory()
d = torch.empty(1024*rows, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
def t(f, n=3):
    best=1e9
    for _ in range(n):
        torch.cuda.synchronize(); t0=time.perf_counter(); f(); torch.cuda.synchronize(); best=min(best,time.perf_counter()-t0)
    return best
gb = nx*rows*8/1e9
for kind,name in ((2,"D2H"),(1,"H2D")):
    def c2d():
        dst,src,dp,sp = (h.data_ptr(), d.data_ptr(), nx*8, 1024*8) if kind==2 else (d.data_ptr(), h.data_ptr(), 1024*8, nx*8)
        assert rt.cudaMemcpy2DAsync(C.c_void_p(dst), C.c_size_t(dp), C.c_void_p(src), C.c_size_t(sp), C.c_size_t(nx*8), C.c_size_t(rows), kind, C.c_void_p(0))==0
    def c1d():
        dst,src = (h.data_ptr(), d.data_ptr()) if kind==2 else (d.data_ptr(), h.data_ptr())
        assert rt.cudaMemcpyAsync(C.c_void_p(dst), C.c_void_p(src), C.c_size_t(nx*rows*8), kind, C.c_void_p(0))==0
    def c2d_chunks():
        R=rows//16
        for c in range(16):
            r0=c*R
            dst,src,dp,sp = (h.data_ptr()+r0*nx*8, d.data_ptr()+r0*1024*8, nx*8, 1024*8) if kind==2 else (d.data_ptr()+r0*1024*8, h.data_ptr()+r0*nx*8, 1024*8, nx*8)
            assert rt.cudaMemcpy2DAsync(C.c_void_p(dst), C.c_size_t(dp), C.c_void_p(src), C.c_size_t(sp), C.c_size_t(nx*8), C.c_size_t(R), kind, C.c_void_p(0))==0
    print(name, "2D 8184B rows (pitch 8192 <-> dense): %.1f GB/s; 1D contiguous: %.1f GB/s; 2D in 16 chunks: %.1f GB/s" % (gb/t(c2d), gb/t(c1d), gb/t(c2d_chunks)), flush=True)
