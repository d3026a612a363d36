// BackendKind::Thomas on the device: per-pole complex tridiagonal solves along
// one axis (reference thomas.cpp:14-160) with the stage epilogues of the split
// step fused into the back substitution (stepper.cpp:221-225, 243-253,
// system_stepper.cpp:89-112).
//
// Q_ell(tau A) b = sum_l 2 Re( r_{ell,l} (tau A - s_l)^{-1} b ) with the LU
// factors of (tau A - s_l) precomputed on the host exactly as factor_pole
// (thomas.cpp:14-29): mul_i = e / piv_{i-1}, piv_i = c - mul_i e.  One thread
// owns one pencil (a line of the field along the axis) and runs the forward
// elimination and the back substitution sequentially; consecutive threads own
// consecutive x positions for the y and z axes (coalesced), consecutive rows
// for the x axis (each thread's 32-byte sectors are re-used from L1 on the next
// three steps).  The forward values live in a [rhs][j][thread] complex scratch
// so a warp's scratch traffic is coalesced on every axis.
//
// Arithmetic follows std::complex<double> operation by operation (products
// and sums as __dmul_rn / __dadd_rn, so nvcc does not fuse them): the y/z
// applies multiply by the host-computed 1/piv (solve_axis_planes), the x
// applies divide by piv (solve_axis_x) with Smith's algorithm.  Whether the
// reference's g++ build contracts its complex products into FMAs depends on
// its flags, so parity is stated as a tolerance (tests/test_gpu_thomas.py).
#pragma once
#include "etd_kernels.cuh"

namespace etd {

enum ThomasEpi { TH_STORE = 0, TH_WHAT = 1, TH_UPDATE = 2 };

struct ThomasArgs {
    const double* in;         // operand stack, stride F
    double* out;              // output stack, stride F
    const double* aux;        // TH_UPDATE: the What stack
    long long F;
    int n;                    // extent along the axis
    long long es;             // element stride along the axis
    long long npencil;        // pencils per field
    long long pin, sa, sb;    // pencil q starts at (q % pin) sa + (q / pin) sb
    int nfields;              // TH_STORE / TH_UPDATE: fields of this launch (field f -> species f % ns)
    int f_first;              // first field of the launch
    int ns;
    int npoles;
    int xdiv;                 // 1: divide by piv (thomas.cpp:42-46); 0: multiply by 1/piv (:69-83)
    int ell;                  // residue set of TH_STORE / TH_UPDATE
    const double2* fac;       // [species][pole][3][n]: mul, piv, 1/piv
    double2 e[2];             // off-diagonal tau off kappa (thomas.cpp:95), per species
    double2 res[2][3][2];     // [species][ell-1][pole]
    double tau;
    double2* scratch;         // [rhs][n][T]
    double* acc;              // [rhs][n][T] partial sums over poles (npoles > 1)
    long long T;              // launched threads
    // TH_WHAT source evaluation (x pencils: row r -> y = r % ny, z = r / ny)
    int ny;
    int gj0, gz0;
    double sp[8];
    const double* sinx;
    const double* siny;
    const double* sinz;
    StepStatus* status;
    int commit;
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                        __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
// Smith's complex division (a + bi) / (c + di)
__device__ __forceinline__ double2 cdiv(double2 n, double2 d) {
    const double a = n.x, b = n.y, c = d.x, dd = d.y;
    if (fabs(c) < fabs(dd)) {
        const double ratio = __ddiv_rn(c, dd);
        const double denom = __dadd_rn(__dmul_rn(c, ratio), dd);
        return make_double2(__ddiv_rn(__dadd_rn(__dmul_rn(a, ratio), b), denom),
                            __ddiv_rn(__dsub_rn(__dmul_rn(b, ratio), a), denom));
    }
    const double ratio = __ddiv_rn(dd, c);
    const double denom = __dadd_rn(__dmul_rn(dd, ratio), c);
    return make_double2(__ddiv_rn(__dadd_rn(__dmul_rn(b, ratio), a), denom),
                        __ddiv_rn(__dsub_rn(b, __dmul_rn(a, ratio)), denom));
}

template <int EPI, int NS, int SK>
__global__ void __launch_bounds__(256, 2) etd_thomas(const ThomasArgs a) {
    constexpr int R = EPI == TH_WHAT ? 2 * NS : 1;
    __shared__ int stop;
    if (threadIdx.x == 0) stop = *reinterpret_cast<volatile int*>(&a.status->fail);
    __syncthreads();
    if (stop) return;
    const long long T = a.T;
    const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long items = EPI == TH_WHAT ? a.npencil : a.npencil * a.nfields;
    const int n = a.n;
    const long long es = a.es;
    const double srcA = (EPI == TH_WHAT && SK == 4) ? exp(-a.sp[0] * (a.status->t + a.tau)) : 0.0;
    int bad = 0, dom = 0;
    for (long long it = tid; it < items; it += T) {
        const int f0 = EPI == TH_WHAT ? 0 : a.f_first + (int)(it / a.npencil);
        const long long q = EPI == TH_WHAT ? it : it % a.npencil;
        const long long base = (q % a.pin) * a.sa + (q / a.pin) * a.sb;
        // right-hand sides: TH_WHAT solves (w1_c, ell 1) and (w2_c, ell 2) for every
        // species c (stack [w1u,(w1v),w2u,(w2v)]); the others one field
        const double* src[R];
        const double2* fc[R];
        double2 e[R], rr[R][2];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int fld = EPI == TH_WHAT ? r : f0;
            const int c = EPI == TH_WHAT ? r % NS : f0 % a.ns;
            const int ell = EPI == TH_WHAT ? (r < NS ? 1 : 2) : a.ell;
            src[r] = a.in + (long long)fld * a.F + base;
            fc[r] = a.fac + (long long)c * a.npoles * 3 * n;
            e[r] = a.e[c];
            rr[r][0] = a.res[c][ell - 1][0];
            rr[r][1] = a.res[c][ell - 1][1];
        }
        for (int l = 0; l < a.npoles; ++l) {
            // forward elimination w_i = b_i - mul_i w_{i-1} (thomas.cpp:38-39, 56-64)
            double2 wp[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                wp[r] = make_double2(__ldg(src[r]), 0.0);
                a.scratch[(long long)r * n * T + tid] = wp[r];
            }
#pragma unroll 4
            for (int j = 1; j < n; ++j) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const double b = __ldg(src[r] + j * es);
                    const double2 m = __ldg(fc[r] + (long long)l * 3 * n + j);
                    const double2 mw = cmul(m, wp[r]);
                    wp[r] = make_double2(__dsub_rn(b, mw.x), -mw.y);
                    a.scratch[((long long)r * n + j) * T + tid] = wp[r];
                }
            }
            // back substitution w_i = (w_i - e w_{i+1}) / piv_i and
            // out_i += 2 Re(r w_i) (thomas.cpp:40-46, 65-84)
            const bool last = l == a.npoles - 1;
            double2 wn[R];
#pragma unroll 2
            for (int j = n - 1; j >= 0; --j) {
                double v[R];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    double2 w = a.scratch[((long long)r * n + j) * T + tid];
                    if (j < n - 1) {
                        const double2 ew = cmul(e[r], wn[r]);
                        w = make_double2(__dsub_rn(w.x, ew.x), __dsub_rn(w.y, ew.y));
                    }
                    const double2* fl = fc[r] + (long long)l * 3 * n;
                    w = a.xdiv ? cdiv(w, __ldg(fl + n + j)) : cmul(w, __ldg(fl + 2 * n + j));
                    wn[r] = w;
                    const double2 rw = cmul(l == 0 ? rr[r][0] : rr[r][1], w);
                    const double c = __dmul_rn(2.0, rw.x);
                    const long long ai = ((long long)r * n + j) * T + tid;
                    v[r] = l == 0 ? __dadd_rn(0.0, c) : __dadd_rn(a.acc[ai], c);
                    if (!last) a.acc[ai] = v[r];
                }
                if (!last) continue;
                const long long o = base + j * es;
                if constexpr (EPI == TH_STORE) {
                    a.out[(long long)f0 * a.F + o] = v[0];
                } else if constexpr (EPI == TH_UPDATE) {
                    // U1 = What + tau Q3(fw) (stepper.cpp:225, 252)
                    const double u1 = __dadd_rn(__ldg(a.aux + (long long)f0 * a.F + o), __dmul_rn(a.tau, v[0]));
                    a.out[(long long)f0 * a.F + o] = u1;
                    bad |= !isfinite(u1);
                } else {
                    // What = Q1(w1) + tau Q2(w2); fw = f(t + tau, What) - w2
                    double W[NS], f[NS];
#pragma unroll
                    for (int c = 0; c < NS; ++c) W[c] = __dadd_rn(v[c], __dmul_rn(a.tau, v[NS + c]));
                    if constexpr (NS == 1) {
                        double ustar = 0.0;
                        if constexpr (SK == 4) {
                            const long long row = q;
                            const int jy = (int)(row % a.ny) + a.gj0, kz = (int)(row / a.ny) + a.gz0;
                            ustar = srcA * (a.sinx[j] * a.siny[jy] * (a.sinz ? a.sinz[kz] : 1.0));
                        }
                        f[0] = src1<SK>(a.sp, W[0], ustar);
                        if constexpr (SK == 3)
                            if (j == 0 && q == 0 && a.gj0 == 0 && a.gz0 == 0)
                                f[0] = __longlong_as_double(0x7ff8000000000000ll);
                        dom |= src_domain_violation<SK>(W[0]);
                    } else {
                        src2<SK>(a.sp, W[0], W[1], f[0], f[1]);
                    }
#pragma unroll
                    for (int c = 0; c < NS; ++c) {
                        bad |= !isfinite(f[c]);
                        a.out[(long long)c * a.F + o] = W[c];
                        a.out[(long long)(NS + c) * a.F + o] =
                            __dsub_rn(f[c], __ldg(a.in + (long long)(NS + c) * a.F + o));
                    }
                }
            }
        }
    }
    const int any_dom = __syncthreads_or(dom), any_bad = __syncthreads_or(bad);
    if (threadIdx.x == 0) {
        if (any_dom || any_bad) {
            int kind = EPI == TH_WHAT ? 2 : EPI == TH_UPDATE ? 3 : 1;
            if (any_dom) kind = 5;
            atomicCAS(&a.status->fail, 0, kind);
        }
        if (EPI == TH_UPDATE && a.commit) {
            __threadfence();
            const unsigned prev = atomicAdd(&a.status->cta_done, 1u);
            if (prev == gridDim.x - 1) {
                __threadfence();
                a.status->cta_done = 0;
                if (*reinterpret_cast<volatile int*>(&a.status->fail) == 0) {
                    const long long nn = a.status->n + 1;
                    a.status->n = nn;
                    a.status->t = (double)nn * a.tau;
                }
            }
        }
    }
}

}  // namespace etd
