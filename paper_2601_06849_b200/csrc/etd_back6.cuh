// etd_back6.cuh — fused second-level backward transform.
//
// The level-2 backward of an axis with n = 4H - 1 (h = 2H) reads the mode
// coefficients in level-2 positions along the axis,
//   [0, H) sigma_c,  [H, 2H) delta_c      (even modes as (X_c + X_{h-1-c}, X_c - X_{h-1-c}))
//   [2H, 3H) Y_lo,   [3H, 4H-1) Y_hi      (odd modes 4c + 1 and 4c + 3)
// and produces the physical pencil g.  For an orbit k < H, c = 2H - 2 - k:
//   o_k  = sum_c P(k, 2c) sigma_c   (k even) | delta_c (k odd)         P(i, 2(h-1-c)) = (-1)^i P(i, 2c)
//   o_c' = the same row for i = c' = 2H - 2 - k (same parity as k)
//   eo_k = sum_c P(k, 4c + 1) Y_lo[c],  ee_k = sum_c P(k, 4c + 3) Y_hi[c]
//   e_k = eo_k + ee_k,  e_c' = eo_k - ee_k      (the odd modes are a DST-I of size 2H - 1)
//   g_k = o_k + e_k,  g_{n-1-k} = o_k - e_k,  g_c' = o_c' + e_c',  g_{n-1-c'} = o_c' - e_c'
// (k = H - 1: c' = k, ee_k = 0 exactly, and the o_c' slot carries the centre
// o_{2H-1} = g_{2H-1}).  The r01 schedule ran this as two launches (the o and the e
// halves into an intermediate stack) and an HBM pass (etd_unfold2) that formed g
// and applied the stage epilogue.  Here one launch contracts all four quarters at
// once — a stage carries four A boxes (the k range of each quarter) — and every
// thread ends up holding whole orbits, so the butterflies and the epilogue run on
// the accumulators: the unfold pass and its HBM round trip disappear.  The DMMA
// sequence of every accumulator is the one of the two-launch path (same operands,
// same k order), so results are bitwise equal to it.
//
// B (matrix G6, etd_plan.cu back6_matrix): 4H rows in blocks of 32; block b has
// parity par = b & 1 and orbit base kb = b >> 1; its four 8-row fragments are the
// types t = 0 (o_k), 1 (o_c'), 2 (eo_k), 3 (ee_k) of k = 16 kb + 2 r + par, r < 8.
// A warp's WN = 64 columns are one block pair (par 0, par 1), so fragment j has
// type j & 3, parity (j >> 2) & 1 and reads A box (type < 2 ? parity : type).  A
// thread (g, l) then holds, per 64-row block pair, the orbits k = 16 kb + 4 l + q,
// q < 4 — four consecutive k, whole orbits, every species of the stack.
#pragma once
#include "etd_kernels.cuh"

namespace etd {

template <int MODE, int S, int BM, int BN, int WARPS_M, int WARPS_N, int STAGES>
struct Back6Cfg {
    static constexpr int BK = 16, AB = 4;
    static constexpr int NW = WARPS_M * WARPS_N, THREADS = 32 * NW;
    static constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;
    static constexpr int MF = WM / 8, NF = WN / 8;
    static constexpr int A1_DBL = S * BM * BK, A_DBL = AB * A1_DBL, B_DBL = BN * BK;
    static constexpr int STAGE_DBL = A_DBL + B_DBL;
    static constexpr uint32_t TX_BYTES = (AB * S * BM + BN) * BK * 8;
    static constexpr int SMEM_BYTES = STAGES * STAGE_DBL * 8 + 1024 + 2 * STAGES * 8 + 64 + 192;  // + CTA trace scratch
    static_assert(WM % 8 == 0 && WN % 64 == 0, "a warp covers whole (par 0, par 1) block pairs");
    static_assert(BM % 16 == 0 && BN % 64 == 0, "cta tile");
};

template <int MODE, int S, int EPI, int SK, int BM, int BN, int WARPS_M, int WARPS_N, int STAGES, int MINB>
__global__ void __launch_bounds__(32 * WARPS_M * WARPS_N, MINB)
    etd_back6(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmA2, const ContractArgs args) {
    static_assert(EPI == EPI_STORE || MODE == 0, "the x stage owns the predictor / update epilogues");
    using C = Back6Cfg<MODE, S, BM, BN, WARPS_M, WARPS_N, STAGES>;
    constexpr int BK = C::BK, MF = C::MF, NF = C::NF;
    (void)tmA2;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    double* smem = reinterpret_cast<double*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_DBL);
    uint64_t* empty = full + STAGES;
    int* cta_flag = reinterpret_cast<int*>(empty + STAGES);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n0 = blockIdx.x * BN;
    const int m0 = (blockIdx.y + args.mtile0) * BM;
    const int outer = blockIdx.z + args.outer0;
    const int H = args.fold_h, n = args.n_axis;
    const int KT = (H + BK - 1) / BK;
    [[maybe_unused]] unsigned long long* tr = reinterpret_cast<unsigned long long*>(cta_flag + 2);
    ETD_TRACE_STAMP(args, tr, 0);

    if (tid == 0) {
        cta_flag[0] = *reinterpret_cast<volatile int*>(&args.status->fail);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], C::NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (cta_flag[0] != 0) return;
    int bad = 0, dom = 0;

    // one TMA per quarter (sigma, delta, Y_lo, Y_hi at axis coordinate q H + k0) and
    // one for the G6 tile; coordinates off the tensor read +0.0
    auto issue = [&](int kt, int stage) {
        double* sA = smem + stage * C::STAGE_DBL;
        double* sB = sA + C::A_DBL;
        mbar_expect_tx(&full[stage], C::TX_BYTES);
        const int k0 = kt * BK;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if constexpr (MODE == 0) tma_load_3d(sA + q * C::A1_DBL, &tmA, &full[stage], k0 + q * H, m0, 0);
            else tma_load_5d(sA + q * C::A1_DBL, &tmA, &full[stage], 0, k0 + q * H, m0 >> 4, outer, 0);
        }
        if constexpr (MODE == 0) tma_load_2d(sB, &tmB, &full[stage], k0, n0);
        else tma_load_3d(sB, &tmB, &full[stage], 0, k0, n0 >> 4);
    };
    if (tid == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
        for (int kt = 0; kt < KT && kt < STAGES; ++kt) issue(kt, kt);
    }

    const int g = lane >> 2, l = lane & 3;
    const int wm0 = (warp / WARPS_N) * C::WM;
    const int wn0 = (warp % WARPS_N) * C::WN;
    double acc[S][MF][NF][2];
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
        for (int i = 0; i < MF; ++i)
#pragma unroll
            for (int j = 0; j < NF; ++j) acc[s][i][j][0] = acc[s][i][j][1] = 0.0;

    // the k permutation of etd_contract (bank-conflict free fragment loads, and the
    // same accumulation order as the two-launch path): FragOffsets below
    // A fragments are double-buffered across steps; B fragments are loaded just in
    // time inside mma() (each feeds S x MF DMMAs), which keeps the 2-CTA/SM class
    // under its 128-register cap
    // (fragment offsets pinned in registers once: FragOffsets, etd_kernels.cuh)
    const FragOffsets<MODE, 0, MF> fo(wm0, wn0, g, l, C::A1_DBL, C::A_DBL);
    // XPAIR (y/z, 16 x per warp): the warp's two M fragments interleave, fragment i row g
    // is x = wm0 + 2 g + i.  Both fragments' A values are then ONE 16-byte LDS (the pair
    // is a swizzle chunk of the [k][16 x] tile: conflict free, a quarter warp reads a whole
    // 128-byte row), and each thread owns two adjacent x of every output: 16-byte stores.
    constexpr bool XPAIR = MODE == 1 && MF == 2;
    int eap[2] = {0, 0};
    if constexpr (XPAIR) {
#pragma unroll
        for (int pp = 0; pp < 2; ++pp) {
            const int kk = 2 * l + pp;
            eap[pp] = pin((wm0 >> 4) * 256 + kk * 16 + ((g ^ (kk & 7)) << 1));
        }
    }
    auto load_frags = [&](int stg, int st, double (&a)[4][S][MF]) {
        const double* sA = smem + stg * C::STAGE_DBL;
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if constexpr (XPAIR) {
                    const double2 v = *reinterpret_cast<const double2*>(sA + q * C::A1_DBL + s * BM * BK +
                                                                        eap[st & 1] + 128 * (st >> 1));
                    a[q][s][0] = v.x;
                    a[q][s][MF - 1] = v.y;
                } else {
#pragma unroll
                    for (int i = 0; i < MF; ++i) a[q][s][i] = sA[q * C::A1_DBL + s * BM * BK + fo.a(st, i)];
                }
            }
    };
    auto mma = [&](int stg, int st, const double (&a)[4][S][MF]) {
        const double* sA = smem + stg * C::STAGE_DBL;
#pragma unroll
        for (int j = 0; j < NF; ++j) {
            const double b = sA[fo.b(st, j)];
            const int t = j & 3, box = t < 2 ? ((j >> 2) & 1) : t;
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int i = 0; i < MF; ++i) dmma884(acc[s][i][j][0], acc[s][i][j][1], a[box][s][i], b);
        }
    };

    double fa[2][4][S][MF];
    int stage = 0;
    uint32_t phase = 0;
    mbar_wait(&full[0], 0);
    ETD_TRACE_STAMP(args, tr, 1);
    load_frags(0, 0, fa[0]);
    for (int kt = 0; kt < KT; ++kt) {
        const int nstage = stage + 1 == STAGES ? 0 : stage + 1;
        const uint32_t nphase = stage + 1 == STAGES ? phase ^ 1 : phase;
#pragma unroll
        for (int st = 0; st < BK / 4; ++st) {
            const int cur = st & 1, nxt = cur ^ 1;
            if (st < BK / 4 - 1) {
                load_frags(stage, st + 1, fa[nxt]);
            } else if (kt + 1 < KT) {
                mbar_wait(&full[nstage], nphase);
                load_frags(nstage, 0, fa[nxt]);
            }
            mma(stage, st, fa[cur]);
            if (st == BK / 4 - 1) {
                // every LDS of this stage is ordered before the TMA refill
                // (consumer_release: generic -> async proxy fence, then arrive)
                consumer_release(&empty[stage], lane);
            }
        }
        if (tid == 0 && kt + STAGES < KT) {
            mbar_wait(&empty[stage], phase);
            issue(kt + STAGES, stage);
        }
        __syncwarp();
        if (kt < 16) ETD_TRACE_STAMP(args, tr, 4 + kt);
        stage = nstage;
        phase = nphase;
    }

    // ===================== orbit epilogue =====================
    ETD_TRACE_STAMP(args, tr, 2);
    double* __restrict__ outp = args.out;
    auto offset = [&](int m, int p) -> long long {
        if constexpr (MODE == 0) return (long long)m * args.pitch + p;
        else return args.zaxis ? (long long)outer * args.pitch + (long long)p * args.plane + m
                               : (long long)outer * args.plane + (long long)p * args.pitch + m;
    };
    const double src_a = SK == 4 ? exp(-args.sp[0] * (args.status->t + args.tau)) : 0.0;
    if constexpr (MODE == 0 && EPI == EPI_WHAT_SRC) {
        // x stage, the predictor: What, f(t + tau, What) with its checks and f - w2's
        // level-2 stack, with the orbit ranges read / written in 16-byte pieces where
        // aligned (as the EPI_UPDATE path below); half A = ranges R0 (k), R1 (n-1-k)
        // from O1 +- e_k, half B = R2 (c), R3 (n-1-c) from O2 +- e_c
#pragma unroll
        for (int i = 0; i < MF; ++i) {
            const int m = m0 + wm0 + i * 8 + g;
            if (m >= args.m_extent) continue;
            const int jj = m % args.ny_local + args.gj0, kz = m / args.ny_local + args.gz0;
#pragma unroll
            for (int bp = 0; bp < NF / 8; ++bp) {
                const int k0 = 16 * ((n0 + wn0) / 64 + bp) + 4 * l;
                if (k0 >= H) continue;
                const bool cen = k0 + 3 == H - 1;
                const long long row = (long long)m * args.pitch;
                const int p1 = n - 1 - k0, p2 = 2 * H - 2 - k0, p3 = 2 * H + k0;
                // w2 at the four ranges, 16-byte where aligned: [s][q]
                auto ldr = [&](const double* a, int R, double (&w)[4]) {
                    if (R == 0) {
                        if constexpr (ETD_BACK6_V4) {
                            ldg_nc_v4(a + k0, w);
                        } else {
                            const double2 x = __ldg(reinterpret_cast<const double2*>(a + k0)),
                                          y = __ldg(reinterpret_cast<const double2*>(a + k0 + 2));
                            w[0] = x.x; w[1] = x.y; w[2] = y.x; w[3] = y.y;
                        }
                    } else if (R == 3 && ETD_BACK6_V4 && !cen) {
                        ldg_nc_v4(a + p3, w);
                    } else if (R == 3) {
                        const double2 x = __ldg(reinterpret_cast<const double2*>(a + p3));
                        w[0] = x.x; w[1] = x.y;
                        if (cen) { w[2] = __ldg(a + p3 + 2); w[3] = 0.0; }
                        else {
                            const double2 y = __ldg(reinterpret_cast<const double2*>(a + p3 + 2));
                            w[2] = y.x; w[3] = y.y;
                        }
                    } else {
                        const int p = R == 1 ? p1 : p2;
                        const double2 x = __ldg(reinterpret_cast<const double2*>(a + p - 2));  // (q2, q1)
                        w[0] = __ldg(a + p);
                        w[1] = x.y;
                        w[2] = x.x;
                        w[3] = __ldg(a + (R == 2 && cen ? 2 * H - 1 : p - 3));
                    }
                };
                auto str = [&](double* o, int R, const double (&v)[4]) {
                    auto st2 = [&](int p, double a, double b) {
                        *reinterpret_cast<double2*>(o + p) = make_double2(a, b);
                    };
                    if (R == 0) {
                        if constexpr (ETD_BACK6_V4) stg_v4(o + k0, v[0], v[1], v[2], v[3]);
                        else { st2(k0, v[0], v[1]); st2(k0 + 2, v[2], v[3]); }
                    } else if (R == 3 && ETD_BACK6_V4 && !cen) {
                        stg_v4(o + p3, v[0], v[1], v[2], v[3]);
                    } else if (R == 3) {
                        st2(p3, v[0], v[1]);
                        if (cen) o[p3 + 2] = v[2];
                        else st2(p3 + 2, v[2], v[3]);
                    } else {
                        const int p = R == 1 ? p1 : p2;
                        st2(p - 2, v[2], v[1]);
                        o[p] = v[0];
                        o[R == 2 && cen ? 2 * H - 1 : p - 3] = v[3];
                    }
                };
                auto fpoint = [&](int x, const double (&gs)[S], double (&fs)[S], bool in) {
                    if constexpr (S == 1) {
                        double ustar = 0.0;
                        if constexpr (SK == 4)
                            ustar = src_a * (args.sinx[x] * args.siny[jj] * (args.sinz ? args.sinz[kz] : 1.0));
                        fs[0] = src1<SK>(args.sp, gs[0], ustar);
                        if constexpr (SK == 3)
                            if (x == 0 && jj == 0 && kz == 0) fs[0] = __longlong_as_double(0x7ff8000000000000ll);
                        bad |= (int)in & (int)!isfinite(fs[0]);
                        dom |= (int)in & src_domain_violation<SK>(gs[0]);
                    } else {
                        src2<SK>(args.sp, gs[0], gs[1], fs[0], fs[1]);
                        bad |= (int)in & (int)!(isfinite(fs[0]) && isfinite(fs[1]));
                    }
                };
                double dk[S][4];
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    const int Ra = 2 * half, Rb = Ra + 1;
                    double ga[S][4], gb[S][4], wa[S][4], wb[S][4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int par = q & 1, e = q >> 1, jb = 8 * bp + 4 * par;
#pragma unroll
                        for (int sp = 0; sp < S; ++sp) {
                            const double EO = acc[sp][i][jb + 2][e], EE = acc[sp][i][jb + 3][e];
                            if (half == 0) {
                                const double O1 = acc[sp][i][jb][e], ek = EO + EE;
                                ga[sp][q] = O1 + ek;
                                gb[sp][q] = O1 - ek;
                            } else {
                                const double O2 = acc[sp][i][jb + 1][e], ec = EO - EE;
                                ga[sp][q] = (cen && q == 3) ? O2 : O2 + ec;
                                gb[sp][q] = O2 - ec;
                            }
                        }
                    }
#pragma unroll
                    for (int sp = 0; sp < S; ++sp) {
                        if (args.aux) {
                            const double* a = args.aux + (long long)sp * args.aux_stride + row;
                            ldr(a, Ra, wa[sp]);
                            ldr(a, Rb, wb[sp]);
                        } else {
#pragma unroll
                            for (int q = 0; q < 4; ++q) wa[sp][q] = wb[sp][q] = 0.0;
                        }
                        double* o = outp + (long long)sp * args.out_stride + row;
                        str(o, Ra, ga[sp]);
                        str(o, Rb, gb[sp]);
                    }
                    // f - w2 at both ranges; stack values of the half
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int k = k0 + q;
                        const bool qc = cen && q == 3;
                        const int xa = half == 0 ? k : (qc ? 2 * H - 1 : 2 * H - 2 - k);
                        const int xb = half == 0 ? n - 1 - k : 2 * H + k;
                        double gsa[S], gsb[S], fa[S], fb[S];
#pragma unroll
                        for (int sp = 0; sp < S; ++sp) { gsa[sp] = ga[sp][q]; gsb[sp] = gb[sp][q]; }
                        fpoint(xa, gsa, fa, true);
                        fpoint(xb, gsb, fb, !(half == 1 && qc));
#pragma unroll
                        for (int sp = 0; sp < S; ++sp) {
                            fa[sp] -= wa[sp][q];
                            fb[sp] -= wb[sp][q];
                            if (half == 0) {
                                ga[sp][q] = fa[sp] + fb[sp];  // s_k (reuses ga)
                                dk[sp][q] = fa[sp] - fb[sp];
                            } else if (qc) {
                                ga[sp][q] = fa[sp] + fa[sp];  // 2 f(2H - 1), the centre of s
                                gb[sp][q] = dk[sp][q] + dk[sp][q];
                            } else {
                                const double sc = fa[sp] + fb[sp], dc = fa[sp] - fb[sp];
                                ga[sp][q] = sc;
                                gb[sp][q] = dk[sp][q] + dc;
                                dk[sp][q] = dk[sp][q] - dc;
                            }
                        }
                    }
                    // level-2 stack positions (fold2_orbit): spos(k) = k/2 (even) | H + k/2 (odd),
                    // spos(c) likewise, 2H + k: d_k + d_c, 3H + k: d_k - d_c
#pragma unroll
                    for (int sp = 0; sp < S; ++sp) {
                        double* fo = args.fout + (long long)sp * args.out_stride + row;
                        auto st2 = [&](int p, double a, double b) {
                            *reinterpret_cast<double2*>(fo + p) = make_double2(a, b);
                        };
                        if (half == 0) {
                            st2(k0 / 2, ga[sp][0], ga[sp][2]);
                            st2(H + k0 / 2, ga[sp][1], ga[sp][3]);
                        } else {
                            st2(H - 2 - k0 / 2, ga[sp][2], ga[sp][0]);           // s_c, c even
                            fo[2 * H - 2 - k0 / 2] = ga[sp][1];                   // s_c, c odd (q = 1)
                            if (cen) fo[2 * H - 1] = ga[sp][3];                   // the centre of s
                            else fo[2 * H - 3 - k0 / 2] = ga[sp][3];              // s_c, c odd (q = 3)
                            if constexpr (ETD_BACK6_V4) {
                                stg_v4(fo + 2 * H + k0, gb[sp][0], gb[sp][1], gb[sp][2], gb[sp][3]);
                            } else {
                                st2(2 * H + k0, gb[sp][0], gb[sp][1]);
                                st2(2 * H + k0 + 2, gb[sp][2], gb[sp][3]);
                            }
                            if (ETD_BACK6_V4 && !cen) {
                                stg_v4(fo + 3 * H + k0, dk[sp][0], dk[sp][1], dk[sp][2], dk[sp][3]);
                            } else {
                                st2(3 * H + k0, dk[sp][0], dk[sp][1]);
                                if (cen) fo[3 * H + k0 + 2] = dk[sp][2];
                                else st2(3 * H + k0 + 2, dk[sp][2], dk[sp][3]);
                            }
                        }
                    }
                }
            }
        }
    } else if constexpr (MODE == 0 && EPI == EPI_UPDATE) {
        // x stage, U1 = What + tau Q3(fw): a thread's four orbits k0 + q (q < 4) are
        // four consecutive positions in each range, so What is read and U1 written in
        // 16-byte pieces where the range is even-aligned (R0 k, R3 2H + k) and as one
        // pair plus two singles where it runs backwards from an odd start (R1 n-1-k,
        // R2 2H-2-k): 10 accesses per species and row instead of 16
#pragma unroll
        for (int i = 0; i < MF; ++i) {
            const int m = m0 + wm0 + i * 8 + g;
            if (m >= args.m_extent) continue;
#pragma unroll
            for (int bp = 0; bp < NF / 8; ++bp) {
                const int k0 = 16 * ((n0 + wn0) / 64 + bp) + 4 * l;
                if (k0 >= H) continue;
                const bool cen = k0 + 3 == H - 1;  // orbit q = 3 is the centre
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    double gq[4][4];  // [q][range]
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int par = q & 1, e = q >> 1, jb = 8 * bp + 4 * par;
                        const double O1 = acc[s][i][jb][e], O2 = acc[s][i][jb + 1][e];
                        const double EO = acc[s][i][jb + 2][e], EE = acc[s][i][jb + 3][e];
                        const double ek = EO + EE, ec = EO - EE;
                        gq[q][0] = O1 + ek;
                        gq[q][1] = O1 - ek;
                        gq[q][2] = (cen && q == 3) ? O2 : O2 + ec;
                        gq[q][3] = O2 - ec;
                    }
                    const double* au = args.aux + (long long)s * args.aux_stride + (long long)m * args.pitch;
                    double* o = outp + (long long)s * args.out_stride + (long long)m * args.pitch;
                    // plain loads (not ld.global.nc): they stay behind the previous species'
                    // stores, so one species is finished -- loads, adds, stores -- before the
                    // next starts; with all 20 loads hoisted ahead of all 20 stores the
                    // launch is 4% slower (r02_experiments.md)
                    auto ld1 = [&](int p) { return au[p]; };
                    auto ld2 = [&](int p) { return *reinterpret_cast<const double2*>(au + p); };
                    auto st2 = [&](int p, double a, double b) { *reinterpret_cast<double2*>(o + p) = make_double2(a, b); };
                    const int p1 = n - 1 - k0, p2 = 2 * H - 2 - k0, p3 = 2 * H + k0;
                    double2 r0a, r0b, r3a, r3b;
                    if constexpr (ETD_BACK6_V4) {
                        double w0[4];
                        ldg_v4(au + k0, w0);
                        r0a = make_double2(w0[0], w0[1]);
                        r0b = make_double2(w0[2], w0[3]);
                        if (!cen) {
                            double w3[4];
                            ldg_v4(au + p3, w3);
                            r3a = make_double2(w3[0], w3[1]);
                            r3b = make_double2(w3[2], w3[3]);
                        } else {
                            r3a = ld2(p3);
                            r3b = make_double2(ld1(p3 + 2), 0.0);
                        }
                    } else {
                        r0a = ld2(k0), r0b = ld2(k0 + 2);
                        r3a = ld2(p3);
                        r3b = cen ? make_double2(ld1(p3 + 2), 0.0) : ld2(p3 + 2);
                    }
                    const double r3c = r3b.x, r3d = r3b.y;
                    const double r1q0 = ld1(p1), r1q3 = ld1(p1 - 3);
                    const double2 r1m = ld2(p1 - 2);  // (q2, q1)
                    const double r2q0 = ld1(p2), r2q3 = ld1(cen ? 2 * H - 1 : p2 - 3);
                    const double2 r2m = ld2(p2 - 2);  // (q2, q1)
                    const double u[4][4] = {{r0a.x + gq[0][0], r1q0 + gq[0][1], r2q0 + gq[0][2], r3a.x + gq[0][3]},
                                            {r0a.y + gq[1][0], r1m.y + gq[1][1], r2m.y + gq[1][2], r3a.y + gq[1][3]},
                                            {r0b.x + gq[2][0], r1m.x + gq[2][1], r2m.x + gq[2][2], r3c + gq[2][3]},
                                            {r0b.y + gq[3][0], r1q3 + gq[3][1], r2q3 + gq[3][2], r3d + gq[3][3]}};
#pragma unroll
                    for (int q = 0; q < 4; ++q)
#pragma unroll
                        for (int R = 0; R < 4; ++R)
                            if (!(cen && q == 3 && R == 3)) bad |= !isfinite(u[q][R]);
                    if constexpr (ETD_BACK6_V4) {
                        stg_v4(o + k0, u[0][0], u[1][0], u[2][0], u[3][0]);
                    } else {
                        st2(k0, u[0][0], u[1][0]);
                        st2(k0 + 2, u[2][0], u[3][0]);
                    }
                    st2(p1 - 2, u[2][1], u[1][1]);
                    o[p1] = u[0][1];
                    o[p1 - 3] = u[3][1];
                    st2(p2 - 2, u[2][2], u[1][2]);
                    o[p2] = u[0][2];
                    o[cen ? 2 * H - 1 : p2 - 3] = u[3][2];
                    if (ETD_BACK6_V4 && !cen) {
                        stg_v4(o + p3, u[0][3], u[1][3], u[2][3], u[3][3]);
                    } else {
                        st2(p3, u[0][3], u[1][3]);
                        if (cen) o[p3 + 2] = u[2][3];
                        else st2(p3 + 2, u[2][3], u[3][3]);
                    }
                }
            }
        }
    } else if constexpr (XPAIR) {
        // y/z store epilogue, two adjacent x per thread (m even; an odd extent's pad
        // column receives the +0.0 its zero A rows produce)
        const int m = m0 + wm0 + 2 * g;
        if (m < args.m_extent) {
#pragma unroll
            for (int bp = 0; bp < NF / 8; ++bp) {
                const int kb = (n0 + wn0) / 64 + bp;
#pragma unroll
                for (int par = 0; par < 2; ++par)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int k = 16 * kb + 4 * l + 2 * e + par;
                        if (k >= H) continue;
                        const int jb = 8 * bp + 4 * par;
                        const bool centre = k == H - 1;
                        const int c = 2 * H - 2 - k;
                        const int np = centre ? 3 : 4;
                        const int pos[4] = {k, n - 1 - k, centre ? 2 * H - 1 : c, n - 1 - c};
#pragma unroll
                        for (int s = 0; s < S; ++s) {
                            double gv[2][4];
#pragma unroll
                            for (int i = 0; i < 2; ++i) {
                                const double O1 = acc[s][i][jb][e], O2 = acc[s][i][jb + 1][e];
                                const double EO = acc[s][i][jb + 2][e], EE = acc[s][i][jb + 3][e];
                                const double ek = EO + EE, ec = EO - EE;
                                gv[i][0] = O1 + ek;
                                gv[i][1] = O1 - ek;
                                gv[i][2] = centre ? O2 : O2 + ec;
                                gv[i][3] = O2 - ec;
                            }
                            double* o = outp + (long long)s * args.out_stride;
#pragma unroll
                            for (int p = 0; p < 4; ++p)
                                if (p < np)
                                    *reinterpret_cast<double2*>(o + offset(m, pos[p])) = make_double2(gv[0][p], gv[1][p]);
                        }
                    }
            }
        }
    } else {
#pragma unroll
    for (int i = 0; i < MF; ++i) {
        const int m = m0 + wm0 + i * 8 + g;
        if (m >= args.m_extent) continue;
#pragma unroll
        for (int bp = 0; bp < NF / 8; ++bp) {
            const int kb = (n0 + wn0) / 64 + bp;
#pragma unroll
            for (int par = 0; par < 2; ++par)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int k = 16 * kb + 4 * l + 2 * e + par;
                    if (k >= H) continue;
                    const int jb = 8 * bp + 4 * par;
                    const bool centre = k == H - 1;
                    const int c = 2 * H - 2 - k;
                    // orbit positions: 0 k, 1 n-1-k, 2 c (centre orbit: 2H-1), 3 n-1-c
                    const int np = centre ? 3 : 4;
                    const int pos[4] = {k, n - 1 - k, centre ? 2 * H - 1 : c, n - 1 - c};
                    double gv[S][4];
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        const double O1 = acc[s][i][jb][e], O2 = acc[s][i][jb + 1][e];
                        const double EO = acc[s][i][jb + 2][e], EE = acc[s][i][jb + 3][e];
                        const double ek = EO + EE, ec = EO - EE;
                        gv[s][0] = O1 + ek;
                        gv[s][1] = O1 - ek;
                        gv[s][2] = centre ? O2 : O2 + ec;
                        gv[s][3] = O2 - ec;
                    }
                    if constexpr (EPI == EPI_STORE) {
#pragma unroll
                        for (int s = 0; s < S; ++s) {
                            double* o = outp + (long long)s * args.out_stride;
#pragma unroll
                            for (int p = 0; p < 4; ++p)
                                if (p < np) o[offset(m, pos[p])] = gv[s][p];
                        }
                    } else if constexpr (EPI == EPI_UPDATE) {
                        // U1 = What + tau Q3(fw) (stepper.cpp:253), checked (fail 3)
                        double w[S][4];
#pragma unroll
                        for (int s = 0; s < S; ++s) {
                            const double* au = args.aux + (long long)s * args.aux_stride;
#pragma unroll
                            for (int p = 0; p < 4; ++p) w[s][p] = p < np ? __ldg(au + offset(m, pos[p])) : 0.0;
                        }
#pragma unroll
                        for (int s = 0; s < S; ++s) {
                            double* o = outp + (long long)s * args.out_stride;
#pragma unroll
                            for (int p = 0; p < 4; ++p) {
                                if (p >= np) break;
                                const double u = w[s][p] + gv[s][p];
                                bad |= !isfinite(u);
                                o[offset(m, pos[p])] = u;
                            }
                        }
                    } else {
                        // EPI_WHAT_SRC: What -> out; f(t + tau, What) at the orbit (fail 2 / 5);
                        // f - w2 (stepper.cpp:252; aux = w2 in physical space) written as
                        // x_fwd_corr's level-2 stack (etd_fold2 positions) -> fout
                        double w2[S][4];
#pragma unroll
                        for (int s = 0; s < S; ++s) {
                            const double* au = args.aux ? args.aux + (long long)s * args.aux_stride : nullptr;
#pragma unroll
                            for (int p = 0; p < 4; ++p) w2[s][p] = (au && p < np) ? __ldg(au + offset(m, pos[p])) : 0.0;
                        }
                        double fv[S][4];
                        const int jj = m % args.ny_local + args.gj0, kz = m / args.ny_local + args.gz0;
#pragma unroll
                        for (int p = 0; p < 4; ++p) {
                            if (p >= np) {
#pragma unroll
                                for (int s = 0; s < S; ++s) fv[s][p] = 0.0;
                                continue;
                            }
                            const int x = pos[p];
                            if constexpr (S == 1) {
                                double ustar = 0.0;
                                if constexpr (SK == 4)
                                    ustar = src_a * (args.sinx[x] * args.siny[jj] * (args.sinz ? args.sinz[kz] : 1.0));
                                fv[0][p] = src1<SK>(args.sp, gv[0][p], ustar);
                                if constexpr (SK == 3)
                                    if (x == 0 && jj == 0 && kz == 0) fv[0][p] = __longlong_as_double(0x7ff8000000000000ll);
                                bad |= !isfinite(fv[0][p]);
                                dom |= src_domain_violation<SK>(gv[0][p]);
                            } else {
                                src2<SK>(args.sp, gv[0][p], gv[1][p], fv[0][p], fv[1][p]);
                                bad |= !(isfinite(fv[0][p]) && isfinite(fv[1][p]));
                            }
#pragma unroll
                            for (int s = 0; s < S; ++s) fv[s][p] -= w2[s][p];
                        }
#pragma unroll
                        for (int s = 0; s < S; ++s) {
                            double* o = outp + (long long)s * args.out_stride;
#pragma unroll
                            for (int p = 0; p < 4; ++p)
                                if (p < np) o[offset(m, pos[p])] = gv[s][p];
                            // the orbit's level-2 stack (fold2_orbit): s_k, s_c, d_k +- d_c,
                            // and for the centre orbit 2 f_centre at 2H - 1
                            double* fo = args.fout + (long long)s * args.out_stride;
                            const double sk = fv[s][0] + fv[s][1], dk = fv[s][0] - fv[s][1];
                            fo[offset(m, fold2_spos(k, H))] = sk;
                            if (centre) {
                                fo[offset(m, 2 * H + k)] = dk + dk;
                                fo[offset(m, 2 * H - 1)] = fv[s][2] + fv[s][2];
                            } else {
                                const double sc = fv[s][2] + fv[s][3], dc = fv[s][2] - fv[s][3];
                                fo[offset(m, fold2_spos(c, H))] = sc;
                                fo[offset(m, 2 * H + k)] = dk + dc;
                                fo[offset(m, 3 * H + k)] = dk - dc;
                            }
                        }
                    }
                }
        }
    }

    }  // generic orbit epilogue

    // ===================== status: abort flag and step commit (as etd_contract) =====================
    const int any_dom = __syncthreads_or(dom);
    const int any_bad = __syncthreads_or(bad);
    ETD_TRACE_STAMP(args, tr, 3);
    ETD_TRACE_FLUSH(args, tr);
    if (tid == 0) {
        if (any_dom || any_bad) {
            int kind = EPI == EPI_WHAT_SRC ? 2 : EPI == EPI_UPDATE ? 3 : 1;
            if (any_dom) kind = 5;
            atomicCAS(&args.status->fail, 0, kind);
        }
        if (EPI == EPI_UPDATE && args.commit) {
            __threadfence();
            const unsigned total = gridDim.x * gridDim.y * gridDim.z;
            const unsigned prev = atomicAdd(&args.status->cta_done, 1u);
            if (prev == total - 1) {
                __threadfence();
                args.status->cta_done = 0;
                if (*reinterpret_cast<volatile int*>(&args.status->fail) == 0) {
                    const long long nn = args.status->n + 1;
                    args.status->n = nn;
                    args.status->t = (double)nn * args.tau;
                }
            }
        }
    }
}

}  // namespace etd
