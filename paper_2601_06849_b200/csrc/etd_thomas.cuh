// BackendKind::Thomas on the device: per-pole complex tridiagonal solves along
// one axis (reference thomas.cpp:14-160) with the stage epilogues of the split
// step fused into the back substitution (stepper.cpp:221-225, 243-253,
// system_stepper.cpp:89-112).
//
// Q_ell(tau A) b = sum_l 2 Re( r_{ell,l} (tau A - s_l)^{-1} b ) with the LU
// factors of (tau A - s_l) precomputed on the host exactly as factor_pole
// (thomas.cpp:14-29): mul_i = e / piv_{i-1}, piv_i = c - mul_i e.
//
// Work split: a CTA of 128 threads owns a tile of 128 pencils (lines of the
// field along the axis), one thread per pencil, and walks the axis with a TMA
// ring of stages (J axis points x 128 pencils x L operands, mbarrier full/empty
// as in the transform kernels), so the sequential recurrences never wait on
// individual global loads:
//   MODE 1 (y/z axes):  5D box {16 x, J, 8 x-blocks, 1, 1}, 128B swizzle
//                       -> [x-block][J][16]   (the pencils are 128 consecutive x)
//   MODE 0 (x axis):    3D box {J=16, 128 rows, 1} per operand, 128B swizzle
//                       -> [row][16]          (the pencils are 128 consecutive rows)
// The stage also carries the rows of mul and 1/piv it needs (bulk copies).
// The forward elimination streams the axis once (all poles together) and keeps
// one checkpoint per chunk of K points; the back substitution streams it again
// in reverse, recomputes each chunk's forward values from its checkpoint in
// registers (the same operations, hence the same bits), finishes every pole of
// the chunk and runs the epilogue.  HBM traffic per point and operand: two reads
// plus the output write; the checkpoints (2 / K of a complex per point) stay
// mostly in L2.  CTAs are persistent over the tiles.
//
// Arithmetic follows std::complex<double> operation by operation (products
// and sums as __dmul_rn / __dadd_rn, so nvcc does not fuse them), with the
// back substitution in the solve_axis_planes form on every axis: multiply by
// the host-computed 1/piv (thomas.cpp:69-83; solve_axis_x divides by piv,
// which differs in the last bit), e w taken componentwise (e is real), and only
// the real part of r w formed.  Whether the reference's g++ build contracts its
// complex products into FMAs depends on its flags, so parity is stated as a
// tolerance (tests/test_gpu_thomas.py).
#pragma once
#include "etd_kernels.cuh"

namespace etd {

enum ThomasEpi { TH_STORE = 0, TH_WHAT = 1, TH_UPDATE = 2 };
// right-hand sides per thread from which the back-substitution chunk is 4 points (else 8)
#ifndef ETD_THOMAS_K4_RHS
#define ETD_THOMAS_K4_RHS 3
#endif
// checkpoint prefetch (unrolled chunk loop) in the coupled predictor too
#ifndef ETD_THOMAS_PREF_WHAT
#define ETD_THOMAS_PREF_WHAT 1
#endif
// ring depth of the x-axis kernels (their stages are L operands wide: 32 KB)
#ifndef ETD_THOMAS_XSTAGES
#define ETD_THOMAS_XSTAGES 3
#endif

struct ThomasArgs {
    double* out;              // output stack, stride F
    long long F;
    int n;                    // extent along the axis
    long long es, so;         // element strides along the axis / the outer index (MODE 1)
    long long pitch;          // row pitch (MODE 0)
    int npen;                 // pencils per outer index: nx (MODE 1) or rows (MODE 0)
    int ptiles;               // 128-pencil tiles per outer index
    int nouter;               // MODE 1: outer extent (nz for y, ny for z); MODE 0: 1
    long long ntiles;         // ptiles * nouter * launch fields
    int f_first;              // first field of the launch (TH_STORE / TH_UPDATE)
    int fin_off;              // TH_UPDATE: stack offset of the fw operands (What at 0)
    int ns;
    int npoles;
    int ell;                  // residue set of TH_STORE / TH_UPDATE
    const double2* fac;       // [species][pole][3][n]: mul, piv, 1/piv
    double2 e[2];             // off-diagonal tau off kappa (thomas.cpp:95), per species
    double2 res[2][3][2];     // [species][ell-1][pole]
    double tau;
    double2* scratch;         // checkpoints [rhs][pole][chunk][CTA][128]
    const double* aux;        // TH_UPDATE: the What fields (the input stack's fields [0, ns))
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

__host__ __device__ constexpr int thomas_rhs(int epi, int ns) { return epi == TH_WHAT ? 2 * ns : 1; }
__host__ __device__ constexpr int thomas_chunk(int rhs) { return rhs >= ETD_THOMAS_K4_RHS ? 4 : 8; }

template <int MODE, int EPI, int NS>
struct ThomasCfg {
    // The coupled two-species predictor (TH_WHAT, NS = 2) splits a pencil over a
    // lane pair, one species per lane (2 rhs per thread instead of 4: half the
    // registers, twice the resident warps); the pair swaps its What values with
    // one shuffle for the coupled source.
    static constexpr bool SPLIT = EPI == TH_WHAT && NS == 2;
    static constexpr int R = SPLIT ? 2 : thomas_rhs(EPI, NS);  // right-hand sides per thread
    static constexpr int K = thomas_chunk(R);              // back-substitution chunk
    static constexpr int T = 128;                          // threads per CTA
    static constexpr int P = SPLIT ? 64 : 128;             // pencils per tile
    static constexpr int J = 16;                           // axis points per stage
    // operands a stage carries (TH_UPDATE reads What straight from global memory in the
    // chunk epilogue: staging it would double the stage and halve the resident CTAs)
    static constexpr int L = MODE == 0 && EPI == TH_WHAT ? 2 * NS : 1;
    static constexpr int STAGES = MODE == 0 ? ETD_THOMAS_XSTAGES : 3;
    static constexpr int OP_DBL = P * J;
    static constexpr int STAGE_DBL = L * OP_DBL;
    static constexpr int NSU = EPI == TH_WHAT ? NS : 1;    // species whose factors a stage carries
    static constexpr int FAC_BYTES = J * 16;               // one factor row slice (mul or 1/piv)
    template <int NP>
    static constexpr int smem_bytes() {
        return STAGES * STAGE_DBL * 8 + STAGES * NSU * NP * 2 * FAC_BYTES + 1024 + 2 * STAGES * 8 + 16;
    }
    static_assert(J % K == 0, "chunks tile the stages");
};

// non-tensor bulk copy global -> shared, completing on an mbarrier
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                        __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

template <int MODE, int EPI, int NS, int SK, int NP>
__global__ void __launch_bounds__(128) etd_thomas(const __grid_constant__ CUtensorMap tm, const ThomasArgs a) {
    using C = ThomasCfg<MODE, EPI, NS>;
    constexpr int R = C::R, K = C::K, J = C::J, L = C::L, S = C::STAGES, P = C::P;
    constexpr bool SPLIT = C::SPLIT;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    double* smem = reinterpret_cast<double*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    // factor row slices per stage: [stage][species u][pole][mul, 1/piv][J]
    double2* fsl = reinterpret_cast<double2*>(smem + S * C::STAGE_DBL);
    constexpr int FS_STAGE = C::NSU * NP * 2 * J;  // double2 per stage
    uint64_t* full = reinterpret_cast<uint64_t*>(fsl + S * FS_STAGE);
    uint64_t* empty = full + S;
    int* flag = reinterpret_cast<int*>(empty + S);
    const int t = threadIdx.x, lane = t & 31;
    if (t == 0) {
        flag[0] = *reinterpret_cast<volatile int*>(&a.status->fail);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], C::T / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (flag[0] != 0) return;

    const int n = a.n;
    const int nt = (n + J - 1) / J, nc = (n + K - 1) / K;
    const int G = gridDim.x;
    const int my_tiles = a.ntiles > (long long)blockIdx.x ? (int)((a.ntiles - blockIdx.x + G - 1) / G) : 0;
    const int per_tile = 2 * nt;               // stages: forward then backward per tile
    const int total = my_tiles * per_tile;
    const double srcA = (EPI == TH_WHAT && SK == 4) ? exp(-a.sp[0] * (a.status->t + a.tau)) : 0.0;

    // ---- producer (thread 0): stage q = (tile i, step s), axis tile forward then reverse
    auto issue = [&](int q) {
        const int slot = q % S;
        const int i = q / per_tile, s = q - i * per_tile;
        const int jt = s < nt ? s : per_tile - 1 - s;
        const long long w = blockIdx.x + (long long)i * G;
        double* dst = smem + slot * C::STAGE_DBL;
        // the forward sweep does not need the 1/piv rows
        const bool fwd = s < nt;
        const int nops = L, nrows = fwd ? 1 : 2;
        mbar_expect_tx(&full[slot], (uint32_t)(nops * C::OP_DBL * 8 + C::NSU * NP * nrows * C::FAC_BYTES));
        const int pb = (int)(w % a.ptiles);
        const int rest = (int)(w / a.ptiles);
        {
            // the stage's rows of mul and 1/piv (the factor arrays are padded past n)
            const int f0 = MODE == 1 ? a.f_first + rest / a.nouter : a.f_first + rest;
#pragma unroll
            for (int u = 0; u < C::NSU; ++u) {
                const int c = EPI == TH_WHAT ? u : f0 % a.ns;
#pragma unroll
                for (int l = 0; l < NP; ++l)
                    for (int m = 0; m < nrows; ++m)
                        bulk_load(fsl + slot * FS_STAGE + ((u * NP + l) * 2 + m) * J,
                                  a.fac + (((long long)c * NP + l) * 3 + 2 * m) * n + jt * J, C::FAC_BYTES,
                                  &full[slot]);
            }
        }
        if constexpr (MODE == 1) {
            const int o = rest % a.nouter, f = a.f_first + rest / a.nouter;
            tma_load_5d(dst, &tm, &full[slot], 0, jt * J, pb * (P / 16), o, f);
        } else {
            const int f = a.f_first + rest;
            for (int op = 0; op < nops; ++op) {
                const int fld = EPI == TH_WHAT ? op : a.fin_off + f;
                tma_load_3d(dst + op * C::OP_DBL, &tm, &full[slot], jt * J, pb * P, fld);
            }
        }
    };
    int issued = 0;
    if (t == 0) {
        tma_prefetch(&tm);
        for (; issued < total && issued < S; ++issued) issue(issued);
    }
    int q = 0;
    auto acquire = [&]() -> const double* {
        const int slot = q % S;
        mbar_wait(&full[slot], (uint32_t)((q / S) & 1));
        return smem + slot * C::STAGE_DBL;
    };
    auto release = [&]() {
        const int slot = q % S;
        consumer_release(&empty[slot], lane);
        ++q;
        // refill the slot of the stage before last (every warp is normally past it);
        // a 2-deep ring refills the slot just released
        if (t == 0)
            for (; issued < total && issued <= q + (S > 2 ? S - 2 : S - 1); ++issued) {
                mbar_wait(&empty[issued % S], (uint32_t)((issued / S - 1) & 1));
                issue(issued);
            }
    };
    // this thread's pencil within the tile, and (SPLIT) its species
    // SPLIT: a warp owns 16 pencils, lanes 0-15 their first species and lanes 16-31 the
    // second, so the 8 lanes of a shared-memory wavefront read 8 consecutive rows of ONE
    // operand tile (8 distinct swizzle chunks).  With the species on adjacent lanes every
    // LDS.128 took 8 wavefronts instead of 4: the two tiles' rows share their banks.
    const int tp = SPLIT ? (t >> 5) * 16 + (lane & 15) : t, sl = SPLIT ? lane >> 4 : 0;
    // operand `op` at axis offset jj of this thread's pencil
    auto rd = [&](const double* st, int op, int jj) -> double {
        if constexpr (MODE == 1) return st[(tp >> 4) * (J * 16) + swz(jj, tp & 15)];
        else return st[op * C::OP_DBL + swz(tp, jj)];
    };
    // N consecutive axis points (jj0 even) of an operand.  MODE 0: a thread's points are
    // consecutive columns of its own row, read as 16-byte pairs -- a pair is one swizzle
    // chunk, so the four rows that share a chunk position fill a 128-byte wavefront
    // (8-byte reads leave half of every wavefront unused: ncu counted as many bank
    // conflicts as useful wavefronts on the x passes)
    auto rdn = [&](const double* st, int op, int jj0, auto& dst) {
        constexpr int N = sizeof(dst) / sizeof(double);
        if constexpr (MODE == 0) {
#pragma unroll
            for (int k2 = 0; k2 < N / 2; ++k2) {
                const double2 pr = *reinterpret_cast<const double2*>(
                    st + op * C::OP_DBL + tp * 16 + ((((jj0 >> 1) + k2) ^ (tp & 7)) << 1));
                dst[2 * k2] = pr.x;
                dst[2 * k2 + 1] = pr.y;
            }
        } else {
#pragma unroll
            for (int k = 0; k < N; ++k) dst[k] = rd(st, op, jj0 + k);
        }
    };
    // operand (= global rhs index for TH_WHAT) of this thread's rhs r
    auto opr = [&](int r) { return EPI == TH_WHAT ? (SPLIT ? r * NS + sl : r) : 0; };
    // checkpoints of this thread: (r, l, c) at cpt[((r * NP + l) * nc + c) * G * P]
    double2* cpt = a.scratch + (long long)blockIdx.x * C::T + t;
    const long long cstr = (long long)G * C::T;

    int bad = 0, dom = 0;
    for (int i = 0; i < my_tiles; ++i) {
        const long long w = blockIdx.x + (long long)i * G;
        const int pb = (int)(w % a.ptiles);
        const int rest = (int)(w / a.ptiles);
        const int pen = pb * P + tp;  // x (MODE 1) or row (MODE 0)
        const bool valid = pen < a.npen;
        int f;
        long long base;
        if constexpr (MODE == 1) {
            f = a.f_first + rest / a.nouter;
            base = pen + (rest % a.nouter) * a.so;
        } else {
            f = a.f_first + rest;
            base = (long long)pen * a.pitch;
        }
        // per rhs: off-diagonal and residues; factor rows come from the stage
        double er[R];
        double2 res[R][NP];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int c = EPI == TH_WHAT ? (SPLIT ? sl : r % NS) : f % a.ns;
            const int ell = EPI == TH_WHAT ? (SPLIT ? r + 1 : (r < NS ? 1 : 2)) : a.ell;
            er[r] = a.e[c].x;
#pragma unroll
            for (int l = 0; l < NP; ++l) res[r][l] = a.res[c][ell - 1][l];
        }
        // factor slice of rhs r, pole l, row m (0 mul, 1 1/piv) in the stage at `st`
        auto fs = [&](const double* st, int r, int l, int m) -> const double2* {
            const int slot = (int)((st - smem) / C::STAGE_DBL);
            const int u = EPI == TH_WHAT ? (SPLIT ? sl : r % NS) : 0;
            return fsl + slot * FS_STAGE + ((u * NP + l) * 2 + m) * J;
        };

        // ---- forward elimination w_i = b_i - mul_i w_{i-1} (thomas.cpp:38-39, 56-64),
        // checkpointing w_{cK-1} before every chunk c
        double2 wp[R][NP];
        constexpr int JP = MODE == 0 ? J : 1;  // the x passes preload a stage's operand values
        auto fwd_point = [&](const double* st, int jj, int j, const double (&bq)[R][JP]) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double b = MODE == 0 ? bq[r][jj % JP] : rd(st, opr(r), jj);
#pragma unroll
                for (int l = 0; l < NP; ++l) {
                    if (j == 0) {
                        wp[r][l] = make_double2(b, 0.0);
                    } else {
                        const double2 mw = cmul(fs(st, r, l, 0)[jj], wp[r][l]);
                        wp[r][l] = make_double2(__dsub_rn(b, mw.x), -mw.y);
                    }
                }
            }
        };
        auto checkpoint = [&](int c) {
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int l = 0; l < NP; ++l) cpt[((long long)(r * NP + l) * nc + c) * cstr] = wp[r][l];
        };
        for (int jt = 0; jt < nt; ++jt) {
            const double* st = acquire();
            const int j0 = jt * J;
            // the stage's operand values (a tile always holds J columns: TMA zero-fills past n)
            double bq[R][JP];
            if constexpr (MODE == 0) {
#pragma unroll
                for (int r = 0; r < R; ++r) rdn(st, opr(r), 0, bq[r]);
            }
            if (jt > 0 && j0 + J <= n) {  // interior stage: no guards
#pragma unroll
                for (int jj = 0; jj < J; ++jj) {
                    if (jj % K == 0) checkpoint((j0 + jj) / K);
                    fwd_point(st, jj, j0 + jj, bq);
                }
            } else {
#pragma unroll
                for (int jj = 0; jj < J; ++jj) {
                    const int j = j0 + jj;
                    if (j < n) {
                        if (jj % K == 0 && j > 0) checkpoint(j / K);
                        fwd_point(st, jj, j, bq);
                    }
                }
            }
            release();
        }

        // ---- back substitution w_i = (w_i - e w_{i+1}) / piv_i, out_i += 2 Re(r w_i)
        // (thomas.cpp:40-46, 65-84), chunk by chunk from the end of the axis: the
        // chunk's forward values are recomputed from its checkpoint (same bits)
        double2 wn[R][NP];
        // Each chunk starts from its checkpoint, an L2 / HBM round trip the recurrence
        // waits for (ncu, config 3: 45% of a pass's stall samples sat on the first use
        // of that load).  PREF: the chunk loop is unrolled over a stage's J / K chunks
        // and chunk cc's checkpoint registers pf[cc] are reloaded, right after their
        // use, with the checkpoint of the same chunk of the next (lower) stage: one
        // stage of lead, no register shuffling (a shifted ring waits on every load it
        // moves: measured slower).  The coupled predictor (TH_WHAT) keeps the plain
        // loop: its stalls move to the shared-memory operand loads and the unrolled
        // body outgrows the instruction cache (x_what 48.2 -> 52.4 ms at config 4).
        constexpr bool PREF = ETD_THOMAS_PREF_WHAT || EPI != TH_WHAT;
        constexpr int NCH = J / K;
        auto cp_load = [&](int c, double2 (&dst)[R][NP]) {
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int l = 0; l < NP; ++l)
                    dst[r][l] = (c > 0 && c < nc) ? cpt[((long long)(r * NP + l) * nc + c) * cstr]
                                                  : make_double2(0.0, 0.0);
        };
        // a chunk's K outputs of one field: 16-byte pairs along an x pencil (the chunk
        // start is even and rows are 16-byte aligned), guarded singles on edge chunks
        auto put = [&](long long fld, int j0, bool edge, const double (&x)[K]) {
            double* o = a.out + fld * a.F + base;
            if constexpr (MODE == 0) {
                if (!edge) {
                    // 32-byte stores (st.global.v4.f64, sm_100): one whole sector each
                    static_assert(K % 4 == 0, "chunks are whole 32-byte pieces");
#pragma unroll
                    for (int k4 = 0; k4 < K / 4; ++k4)
                        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(o + j0 + 4 * k4), "d"(x[4 * k4]),
                                     "d"(x[4 * k4 + 1]), "d"(x[4 * k4 + 2]), "d"(x[4 * k4 + 3])
                                     : "memory");
                    return;
                }
            }
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int j = j0 + k;
                if (edge && j >= n) continue;
                o[MODE == 0 ? (long long)j : j * a.es] = x[k];
            }
        };
        auto chunk = [&](const double* st, int jt, int cc, const double2 (&cp0)[R][NP]) {
                const int j0 = jt * J + cc * K, c = j0 / K;
                if (j0 >= n) return;
                const bool edge = c == 0 || j0 + K >= n;  // first chunk, or holds j = n - 1
                constexpr int KP = MODE == 0 ? K : 1;
                double bq[R][KP];
                if constexpr (MODE == 0) {
#pragma unroll
                    for (int r = 0; r < R; ++r) rdn(st, opr(r), cc * K, bq[r]);
                }
                [[maybe_unused]] double aq[K];  // TH_UPDATE: What
                if constexpr (EPI == TH_UPDATE) {
                    // issued here, used after the chunk's recurrences
                    const double* w = a.aux + (long long)f * a.F + base + (MODE == 0 ? (long long)j0 : j0 * a.es);
                    if (MODE == 0 && !edge && valid) {
#pragma unroll
                        for (int k4 = 0; k4 < K / 4; ++k4)
                            asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                                         : "=d"(aq[4 * k4]), "=d"(aq[4 * k4 + 1]), "=d"(aq[4 * k4 + 2]), "=d"(aq[4 * k4 + 3])
                                         : "l"(w + 4 * k4));
                    } else {
#pragma unroll
                        for (int k = 0; k < K; ++k)
                            aq[k] = (valid && j0 + k < n) ? __ldg(w + (MODE == 0 ? (long long)k : k * a.es)) : 0.0;
                    }
                }
                double v[R][K];
#pragma unroll
                for (int l = 0; l < NP; ++l) {
                    double2 wv[R][K];
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        double2 prev = cp0[r][l];
#pragma unroll
                        for (int k = 0; k < K; ++k) {
                            const int j = j0 + k;
                            if (edge && j >= n) break;
                            const double b = MODE == 0 ? bq[r][k % KP] : rd(st, opr(r), cc * K + k);
                            if (edge && j == 0) {
                                prev = make_double2(b, 0.0);
                            } else {
                                const double2 mw = cmul(fs(st, r, l, 0)[cc * K + k], prev);
                                prev = make_double2(__dsub_rn(b, mw.x), -mw.y);
                            }
                            wv[r][k] = prev;
                        }
                    }
#pragma unroll
                    for (int k = K - 1; k >= 0; --k) {
                        const int j = j0 + k;
                        if (edge && j >= n) continue;
#pragma unroll
                        for (int r = 0; r < R; ++r) {
                            double2 x = wv[r][k];
                            if (!edge || j < n - 1) {
                                // e is real (tau off kappa): e w componentwise
                                x = make_double2(__dsub_rn(x.x, __dmul_rn(er[r], wn[r][l].x)),
                                                 __dsub_rn(x.y, __dmul_rn(er[r], wn[r][l].y)));
                            }
                            x = cmul(x, fs(st, r, l, 1)[cc * K + k]);
                            wn[r][l] = x;
                            const double con = __dmul_rn(
                                2.0, __dsub_rn(__dmul_rn(res[r][l].x, x.x), __dmul_rn(res[r][l].y, x.y)));
                            v[r][k] = l == 0 ? __dadd_rn(0.0, con) : __dadd_rn(v[r][k], con);
                        }
                    }
                }
                if constexpr (SPLIT) {
                    // What of this lane's species; the pair swaps them for f(t + tau, What)
                    // (all lanes of the warp take this path: same chunk, same guards)
                    double o0[K], o1[K];
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        const int j = j0 + k;
                        o0[k] = o1[k] = 0.0;
                        if (edge && j >= n) continue;
                        const double Wm = __dadd_rn(v[0][k], __dmul_rn(a.tau, v[1][k]));
                        const double Wo = __shfl_xor_sync(0xffffffffu, Wm, 16);
                        if (!valid) continue;
                        const double Wu = sl == 0 ? Wm : Wo, Wv = sl == 0 ? Wo : Wm;
                        double fu, fv;
                        src2<SK>(a.sp, Wu, Wv, fu, fv);
                        const double fm = sl == 0 ? fu : fv;
                        bad |= !isfinite(fm);
                        o0[k] = Wm;
                        o1[k] = __dsub_rn(fm, MODE == 0 ? bq[1][k % KP] : 0.0);  // rhs 1 = w2 of this species
                    }
                    if (!valid) return;
                    put(sl, j0, edge, o0);
                    put(NS + sl, j0, edge, o1);
                    return;
                }
                if (!valid) return;
                if constexpr (EPI == TH_STORE) {
                    put(f, j0, edge, v[0]);
                } else if constexpr (EPI == TH_UPDATE) {
                    // U1 = What + tau Q3(fw) (stepper.cpp:225, 252)
                    double u1[K];
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        u1[k] = 0.0;
                        if (edge && j0 + k >= n) continue;
                        u1[k] = __dadd_rn(aq[k], __dmul_rn(a.tau, v[0][k]));
                        bad |= !isfinite(u1[k]);
                    }
                    put(f, j0, edge, u1);
                } else if constexpr (!SPLIT) {
                    // What = Q1(w1) + tau Q2(w2); fw = f(t + tau, What) - w2
                    double Wk[NS][K], gk[NS][K];
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        const int j = j0 + k;
#pragma unroll
                        for (int s = 0; s < NS; ++s) Wk[s][k] = gk[s][k] = 0.0;
                        if (edge && j >= n) continue;
                        double W[NS], fv[NS];
#pragma unroll
                        for (int s = 0; s < NS; ++s) W[s] = __dadd_rn(v[s][k], __dmul_rn(a.tau, v[NS + s][k]));
                        if constexpr (NS == 1) {
                            double ustar = 0.0;
                            if constexpr (SK == 4) {
                                const int jy = pen % a.ny + a.gj0, kz = pen / a.ny + a.gz0;
                                ustar = srcA * (a.sinx[j] * a.siny[jy] * (a.sinz ? a.sinz[kz] : 1.0));
                            }
                            fv[0] = src1<SK>(a.sp, W[0], ustar);
                            if constexpr (SK == 3)
                                if (j == 0 && pen == 0 && a.gj0 == 0 && a.gz0 == 0)
                                    fv[0] = __longlong_as_double(0x7ff8000000000000ll);
                            dom |= src_domain_violation<SK>(W[0]);
                        } else {
                            src2<SK>(a.sp, W[0], W[1], fv[0], fv[1]);
                        }
#pragma unroll
                        for (int s = 0; s < NS; ++s) {
                            bad |= !isfinite(fv[s]);
                            Wk[s][k] = W[s];
                            gk[s][k] = __dsub_rn(fv[s], MODE == 0 ? bq[NS + s][k % KP] : 0.0);  // rhs NS + s = w2
                        }
                    }
#pragma unroll
                    for (int s = 0; s < NS; ++s) {
                        put(s, j0, edge, Wk[s]);
                        put(NS + s, j0, edge, gk[s]);
                    }
                }
        };
        double2 pf[PREF ? NCH : 1][R][NP];
        if constexpr (PREF) {
#pragma unroll
            for (int cc = 0; cc < NCH; ++cc) cp_load((nt - 1) * NCH + cc, pf[cc]);
        }
        for (int jt = nt - 1; jt >= 0; --jt) {
            const double* st = acquire();
            if constexpr (PREF) {
#pragma unroll
                for (int cc = NCH - 1; cc >= 0; --cc) {
                    double2 cp0[R][NP];
#pragma unroll
                    for (int r = 0; r < R; ++r)
#pragma unroll
                        for (int l = 0; l < NP; ++l) cp0[r][l] = pf[cc][r][l];
                    cp_load(jt * NCH + cc - NCH, pf[cc]);
                    chunk(st, jt, cc, cp0);
                }
            } else {
#pragma unroll 1
                for (int cc = NCH - 1; cc >= 0; --cc) {
                    cp_load(jt * NCH + cc, pf[0]);
                    chunk(st, jt, cc, pf[0]);
                }
            }
            release();
        }
    }

    const int any_dom = __syncthreads_or(dom), any_bad = __syncthreads_or(bad);
    if (t == 0) {
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
