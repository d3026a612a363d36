// FP64 throughput microbenchmark for B200 (sm_100a).
//
// Measures the chip-wide FP64 rate of the two instruction paths the
// eigenbasis-transform kernels can use:
//   * DMMA  (mma.sync.aligned.m8n8k4 / m16n8k{4,8,16} .f64)  -> SASS DMMA.8x8x4
//   * DFMA  (scalar fma.rn.f64)                                -> SASS DFMA
// and the single-warp DMMA dependency latency.  The result is the FP64 peak
// that roofline.peak in bench.py is quoted against (MEASURED_PEAKS.json has no
// FP64 entry).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    std::fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); std::exit(1);} } while (0)

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma1684(double* c, double a0, double a1, double b) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(b));
}
__device__ __forceinline__ void dmma1688(double* c, const double* a, const double* b) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

template <int NACC>
__global__ void k_dmma884(double* out, int iters, double seed) {
    double c[NACC][2];
    double a = seed * (threadIdx.x + 1), b = seed * 0.5;
#pragma unroll
    for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) dmma884(c[i][0], c[i][1], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void k_dmma1684(double* out, int iters, double seed) {
    double c[NACC][4];
    double a0 = seed * (threadIdx.x + 1), a1 = seed * 0.25, b = seed * 0.5;
#pragma unroll
    for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) dmma1684(c[i], a0, a1, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 12345.678) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void k_dmma1688(double* out, int iters, double seed) {
    double c[NACC][4];
    double a[4], b[2];
    for (int j = 0; j < 4; ++j) a[j] = seed * (threadIdx.x + j);
    b[0] = seed; b[1] = seed * 2;
#pragma unroll
    for (int i = 0; i < NACC; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) dmma1688(c[i], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 12345.678) out[threadIdx.x] = s;
}

template <int NCH>
__global__ void k_dfma(double* out, int iters, double seed) {
    double c[NCH];
    const double a = 1.0000001, b = seed * 1e-9;
#pragma unroll
    for (int i = 0; i < NCH; ++i) c[i] = seed * (i + threadIdx.x);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NCH; ++i) c[i] = fma(c[i], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < NCH; ++i) s += c[i];
    if (s == 12345.678) out[threadIdx.x] = s;
}

template <typename K>
static double time_kernel(K kern, int blocks, int threads, int iters, double* out) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    for (int w = 0; w < 2; ++w) kern<<<blocks, threads>>>(out, iters, 1.0);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(e0));
        kern<<<blocks, threads>>>(out, iters, 1.0);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
    }
    CK(cudaEventDestroy(e0)); CK(cudaEventDestroy(e1));
    return best * 1e-3;
}

int main(int argc, char** argv) {
    int dev = 0; CK(cudaSetDevice(dev));
    cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
    int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    std::printf("{\"device\": \"%s\", \"sms\": %d, \"clock_mhz_attr\": %d}\n", p.name, p.multiProcessorCount, clk_khz / 1000);
    double* out; CK(cudaMalloc(&out, 4096 * sizeof(double)));
    const int sms = p.multiProcessorCount;
    const int iters = argc > 1 ? std::atoi(argv[1]) : 20000;

    // chip-wide rate at several warps/SM
    for (int wps : {4, 8, 16, 32}) {
        const int threads = 32 * (wps > 16 ? 16 : wps);
        const int blocks = sms * (wps > 16 ? wps / 16 : 1);
        double t = time_kernel(k_dmma884<8>, blocks, threads, iters, out);
        double fl = double(blocks) * (threads / 32) * iters * 8 * 512.0;
        std::printf("{\"kind\": \"dmma_m8n8k4\", \"warps_per_sm\": %d, \"acc\": 8, \"tflops\": %.3f}\n", wps, fl / t * 1e-12);
    }
    for (int wps : {4, 8, 16}) {
        const int threads = 32 * wps, blocks = sms;
        double t = time_kernel(k_dmma1684<8>, blocks, threads, iters, out);
        double fl = double(blocks) * wps * iters * 8 * 1024.0;
        std::printf("{\"kind\": \"dmma_m16n8k4\", \"warps_per_sm\": %d, \"acc\": 8, \"tflops\": %.3f}\n", wps, fl / t * 1e-12);
        t = time_kernel(k_dmma1688<8>, blocks, threads, iters / 2, out);
        fl = double(blocks) * wps * (iters / 2) * 8 * 2048.0;
        std::printf("{\"kind\": \"dmma_m16n8k8\", \"warps_per_sm\": %d, \"acc\": 8, \"tflops\": %.3f}\n", wps, fl / t * 1e-12);
    }
    for (int wps : {8, 16, 32}) {
        const int threads = 32 * (wps > 16 ? 16 : wps);
        const int blocks = sms * (wps > 16 ? wps / 16 : 1);
        double t = time_kernel(k_dfma<8>, blocks, threads, iters, out);
        double fl = double(blocks) * threads * iters * 8 * 2.0;
        std::printf("{\"kind\": \"dfma\", \"warps_per_sm\": %d, \"chains\": 8, \"tflops\": %.3f}\n", wps, fl / t * 1e-12);
    }
    // single-warp dependent-chain latency (one accumulator)
    {
        double t = time_kernel(k_dmma884<1>, 1, 32, iters, out);
        std::printf("{\"kind\": \"dmma_m8n8k4_latency\", \"ns_per_dep_mma\": %.3f}\n", t / iters * 1e9);
        t = time_kernel(k_dmma884<4>, 1, 32, iters, out);
        std::printf("{\"kind\": \"dmma_m8n8k4_1warp_4acc\", \"ns_per_mma\": %.3f}\n", t / iters / 4 * 1e9);
        t = time_kernel(k_dfma<1>, 1, 32, iters, out);
        std::printf("{\"kind\": \"dfma_latency\", \"ns_per_dep_fma\": %.3f}\n", t / iters * 1e9);
    }
    // sustained: a long DMMA run (~several seconds) to see the power-capped rate
    {
        const int wps = 16, threads = 512, blocks = sms;
        const int long_iters = iters * 40;
        double t = time_kernel(k_dmma884<8>, blocks, threads, long_iters, out);
        double fl = double(blocks) * wps * long_iters * 8 * 512.0;
        std::printf("{\"kind\": \"dmma_m8n8k4_sustained\", \"seconds\": %.3f, \"tflops\": %.3f}\n", t, fl / t * 1e-12);
    }
    CK(cudaFree(out));
    return 0;
}
