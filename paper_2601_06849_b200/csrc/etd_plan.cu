// etd_plan.cu — host orchestration of the B200 ETD2RK-DS step and the C-ABI
// (include/etd_b200.h).  One handle = one plan (reference StepperPlan /
// SystemPlan, stepper.hpp:35-56,91-105) + its device-resident state.
//
// Step schedule (3D; 13 transforms, PAPER Algorithm 2 / stepper.cpp:233-257,
// system_stepper.cpp:74-114), ns = number of species, F = one padded field:
//   1 z_fwd_src  [U(,V)] --f--> [U,(V),fU,(fV)] x Pz^T, * 2 d1z  -> Z
//   2 z_back     Z x Pz                                           -> W
//   3 y_fwd      W x Py^T, * 2 d1y                                -> Z
//   4 y_back     Z x Py                                 -> W = [w1.., w2..]
//   5 x_fwd_mix  W x Px^T: Z[c] = 2d1 w1b + 2tau d2 w2b, Z[ns+c] = w2b
//   6 x_back_src Z[0:ns] x Px: W[c] = What, W[ns+c] = f(What)   (check t+tau)
//   7 x_fwd_corr W[ns:] x Px^T: Z[c] = (. - w2b) 2 tau d3
//   8 x_back_upd Z[0:ns] x Px + What -> state'                   (check, commit)
// 2D replaces 1-4 by y_fwd_src + y_back (9 transforms, Algorithm 1 /
// stepper.cpp:182-229).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <sys/mman.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <numbers>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/etd_b200.h"
#include "etd_registry.cuh"
#include "etd_thomas.cuh"
#include "etd_setup.hpp"

namespace etd {

struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };
struct AbortError : std::runtime_error {
    AbortError(const std::string& m, double t_, long s_) : std::runtime_error(m), t(t_), step(s_) {}
    double t;
    long step;
};
struct NoDevice : std::runtime_error { using std::runtime_error::runtime_error; };

#define ETD_CK(x)                                                                              \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess)                                                                 \
            throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));                 \
    } while (0)

// ------------------------------------------------------------ tensor maps
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        ETD_CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// FP64 tiled map, 128B swizzle, OOB elements read as +0.0 (never touch pads).
static CUtensorMap make_map(const double* base, int rank, const unsigned long long* dims,
                            const unsigned long long* strides_elems, const unsigned* box,
                            CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B) {
    CUtensorMap m;
    cuuint64_t gd[5], gs[4];
    cuuint32_t bx[5], es[5];
    for (int i = 0; i < rank; ++i) {
        gd[i] = dims[i];
        bx[i] = box[i];
        es[i] = 1;
    }
    for (int i = 0; i < rank - 1; ++i) gs[i] = strides_elems[i] * sizeof(double);
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<double*>(base), gd, gs,
                             bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    return m;
}

// fold: 0 dense, 1-4 parity split (etd_kernels.cuh).  Kernels that evaluate the
// source are instantiated per source kind; every other kernel ignores sk.
static KernelSpec pick(int mode, int S, int epi, bool pro, int sk = 0, int tile = 0, int fold = 0) {
    const bool uses_src = pro || epi == EPI_WHAT_SRC;
    if (!uses_src) sk = 0;
    if (fold == 6) {
        if (pro || tile == 1) throw ConfigError("no fused level-2 backward variant for this tile");
        return pick_back6(mode, S, epi, sk, tile);
    }
    return fold ? pick_fold(mode, S, epi, sk, tile, fold) : pick_dense(mode, S, epi, pro, sk, tile);
}

static const void* pick_unfold(int sk, int uf) {
#define ETD_UF(K)                                                                                          \
    case K:                                                                                                \
        return uf == UF_WHAT_SRC ? reinterpret_cast<const void*>(etd_unfold2<K, UF_WHAT_SRC>)              \
               : uf == UF_UPDATE ? reinterpret_cast<const void*>(etd_unfold2<K, UF_UPDATE>)                 \
                                 : reinterpret_cast<const void*>(etd_unfold2<K, UF_STORE>);
    switch (sk) {
        ETD_UF(0) ETD_UF(1) ETD_UF(2) ETD_UF(3) ETD_UF(4) ETD_UF(5) ETD_UF(10) ETD_UF(11) ETD_UF(12) ETD_UF(13)
    default: throw ConfigError("unknown source kind");
    }
#undef ETD_UF
}

// level-2 source pass (etd_source_l2): variant v = 1 (16-byte x pairs, 3 blocks/SM),
// 2 (one x per thread, 4 blocks/SM); 3 / 4 the same with the outer index fastest;
// 5 x pairs, 2 blocks, outer fastest
template <int SK>
static const void* pick_source_l2_sk(int ns, int v) {
#define ETD_SL2(NS)                                                                                   \
    (v == 1   ? reinterpret_cast<const void*>(etd_source_l2<SK, NS, 2, 3, false>)                      \
     : v == 2 ? reinterpret_cast<const void*>(etd_source_l2<SK, NS, 1, 4, false>)                      \
     : v == 3 ? reinterpret_cast<const void*>(etd_source_l2<SK, NS, 2, 3, true>)                       \
     : v == 4 ? reinterpret_cast<const void*>(etd_source_l2<SK, NS, 1, 4, true>)                       \
              : reinterpret_cast<const void*>(etd_source_l2<SK, NS, 2, 2, true>))
    return ns == 1 ? ETD_SL2(1) : ETD_SL2(2);
#undef ETD_SL2
}

// y/z fused backward launches: one field per launch (S = 1 tiles, XPAIR fragment interleave,
// etd_back6.cuh) unless ETD_BACK6_XPAIR=0 (S = 4 stacks as two S = 2 launches; A/B)
static bool back6_xpair() {
    const char* e = std::getenv("ETD_BACK6_XPAIR");
    return !(e && atoi(e) == 0);
}

static int source_l2_variant() {
    const char* e = getenv("ETD_SRC_L2");
    return e ? atoi(e) : 3;
}

static const void* pick_source(int sk, int ns = 0, bool fold2 = false) {
    const int v = source_l2_variant();
    if (fold2 && v > 0) {
        switch (sk) {
        case 0: return pick_source_l2_sk<0>(ns, v);
        case 1: return pick_source_l2_sk<1>(ns, v);
        case 2: return pick_source_l2_sk<2>(ns, v);
        case 3: return pick_source_l2_sk<3>(ns, v);
        case 4: return pick_source_l2_sk<4>(ns, v);
        case 5: return pick_source_l2_sk<5>(ns, v);
        case 10: return pick_source_l2_sk<10>(ns, v);
        case 11: return pick_source_l2_sk<11>(ns, v);
        case 12: return pick_source_l2_sk<12>(ns, v);
        case 13: return pick_source_l2_sk<13>(ns, v);
        default: throw ConfigError("unknown source kind");
        }
    }
    switch (sk) {
    case 0: return reinterpret_cast<const void*>(etd_source<0>);
    case 1: return reinterpret_cast<const void*>(etd_source<1>);
    case 2: return reinterpret_cast<const void*>(etd_source<2>);
    case 3: return reinterpret_cast<const void*>(etd_source<3>);
    case 4: return reinterpret_cast<const void*>(etd_source<4>);
    case 5: return reinterpret_cast<const void*>(etd_source<5>);
    case 10: return reinterpret_cast<const void*>(etd_source<10>);
    case 11: return reinterpret_cast<const void*>(etd_source<11>);
    case 12: return reinterpret_cast<const void*>(etd_source<12>);
    case 13: return reinterpret_cast<const void*>(etd_source<13>);
    default: throw ConfigError("unknown source kind");
    }
}

// Thomas kernels: MODE 1 (y/z) only stores (the z/y filters); MODE 0 (x) runs
// every epilogue, and only TH_WHAT evaluates a source.
struct ThomasSpec {
    const void* fn = nullptr;
    int smem = 0;
    int occ = 0;  // resident CTAs per SM (set once the smem attribute is applied)
    int pencils = 128;  // pencils per tile (64 for the lane-pair split predictor)
};
template <int MODE, int EPI, int NS, int SK>
static ThomasSpec thomas_spec(int np) {
    const void* fn = np == 1 ? reinterpret_cast<const void*>(etd_thomas<MODE, EPI, NS, SK, 1>)
                             : reinterpret_cast<const void*>(etd_thomas<MODE, EPI, NS, SK, 2>);
    const int smem = np == 1 ? ThomasCfg<MODE, EPI, NS>::template smem_bytes<1>()
                             : ThomasCfg<MODE, EPI, NS>::template smem_bytes<2>();
    return {fn, smem, 0, ThomasCfg<MODE, EPI, NS>::P};
}
template <int MODE, int EPI, int NS>
static ThomasSpec thomas_sk(int sk, int np) {
    if constexpr (EPI != TH_WHAT) {
        return thomas_spec<MODE, EPI, NS, 0>(np);
    } else if constexpr (NS == 1) {
        switch (sk) {
        case 0: return thomas_spec<MODE, EPI, 1, 0>(np);
        case 1: return thomas_spec<MODE, EPI, 1, 1>(np);
        case 2: return thomas_spec<MODE, EPI, 1, 2>(np);
        case 3: return thomas_spec<MODE, EPI, 1, 3>(np);
        case 4: return thomas_spec<MODE, EPI, 1, 4>(np);
        case 5: return thomas_spec<MODE, EPI, 1, 5>(np);
        }
    } else {
        switch (sk) {
        case 0: return thomas_spec<MODE, EPI, 2, 0>(np);
        case 10: return thomas_spec<MODE, EPI, 2, 10>(np);
        case 11: return thomas_spec<MODE, EPI, 2, 11>(np);
        case 12: return thomas_spec<MODE, EPI, 2, 12>(np);
        case 13: return thomas_spec<MODE, EPI, 2, 13>(np);
        }
    }
    throw ConfigError("unknown source kind");
}
static ThomasSpec pick_thomas(int mode, int epi, int ns, int sk, int np) {
    if (np != 1 && np != 2) throw ConfigError("Thomas backend: 1 or 2 poles");
    ThomasSpec k;
    if (mode == 1) {
        if (epi != TH_STORE) throw ConfigError("Thomas y/z passes only store");
        k = ns == 1 ? thomas_sk<1, TH_STORE, 1>(sk, np) : thomas_sk<1, TH_STORE, 2>(sk, np);
    } else if (epi == TH_STORE) {
        k = ns == 1 ? thomas_sk<0, TH_STORE, 1>(sk, np) : thomas_sk<0, TH_STORE, 2>(sk, np);
    } else if (epi == TH_WHAT) {
        k = ns == 1 ? thomas_sk<0, TH_WHAT, 1>(sk, np) : thomas_sk<0, TH_WHAT, 2>(sk, np);
    } else {
        k = ns == 1 ? thomas_sk<0, TH_UPDATE, 1>(sk, np) : thomas_sk<0, TH_UPDATE, 2>(sk, np);
    }
    // large dynamic shared memory + occupancy, once per kernel
    static std::vector<std::pair<const void*, int>> done;
    for (auto& dn : done)
        if (dn.first == k.fn) {
            k.occ = dn.second;
            return k;
        }
    ETD_CK(cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, k.smem));
    ETD_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&k.occ, k.fn, 128, k.smem));
    if (k.occ < 1) throw CudaError("Thomas kernel does not fit on an SM");
    done.push_back({k.fn, k.occ});
    return k;
}

// ------------------------------------------------------------ NCCL (dlopen'd)
// The extension does not link NCCL: single-GPU users and CPU tests never load
// it.  Sharded plans resolve it at etd_create (torch's bundled libnccl.so.2
// when torch is already loaded, else the system one).
struct Nccl {
    using ncclComm_t = void*;
    int (*GetUniqueId)(ncclUniqueId*) = nullptr;
    int (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    int (*CommDestroy)(ncclComm_t) = nullptr;
    int (*CommCount)(ncclComm_t, int*) = nullptr;
    int (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
    bool ok = false;

    static Nccl& get() {
        static Nccl n;
        if (!n.ok) {
            void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
            if (!h) throw CudaError("libnccl.so.2 not found (needed for z-slab sharding)");
            auto sym = [&](const char* s) {
                void* f = dlsym(h, s);
                if (!f) throw CudaError(std::string("NCCL symbol missing: ") + s);
                return f;
            };
            n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
            n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
            n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
            n.CommCount = reinterpret_cast<decltype(n.CommCount)>(sym("ncclCommCount"));
            n.Send = reinterpret_cast<decltype(n.Send)>(sym("ncclSend"));
            n.Recv = reinterpret_cast<decltype(n.Recv)>(sym("ncclRecv"));
            n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
            n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
            n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
            n.ok = true;
        }
        return n;
    }
    void check(int r, const char* what) const {
        if (r != 0) throw CudaError(std::string(what) + ": " + (GetErrorString ? GetErrorString(r) : "nccl error"));
    }
};

// ------------------------------------------------------------ the plan
struct Launch {
    std::string name;
    int mode = 0, S = 1, epi = 0, tile = 0, fold = 0;
    bool pro = false;
    KernelSpec k;
    dim3 grid;
    CUtensorMap tmA, tmB, tmA2;  // tmA2: FOLD 3's x-reversed operand (= tmA otherwise)
    ContractArgs args;
    double flops = 0, bytes = 0;
    double dense_flops = 0;  // the same transform as a dense n x n contraction
};

// A piece of an exchange: `bytes` at `ptr` to (send) or from (recv) rank `peer`.
struct Piece {
    int peer;
    void* ptr;
    size_t bytes;
};

struct Op {
    enum Kind { KERNEL, SOURCE, COPY2D, EXCHANGE, FAILCODE, COMMIT, THOMAS, NOP, FOLD, UNFOLD, ZYFOLD } kind = KERNEL;
    // sharded steps: 1 = run on the communication stream; events (indices into
    // Plan::sev) waited on before / recorded after the op (ignored by virtual ranks)
    int strm = 0, wait_ev = -1, rec_ev = -1;
    Launch L;                                    // KERNEL (and SOURCE/THOMAS: name/flops/bytes)
    SourceArgs sargs{};                          // SOURCE
    ThomasArgs targs{};                          // THOMAS
    Fold2Args fargs{};                           // FOLD (second-level split stack, etd_fold2)
    Unfold2Args uargs{};                         // UNFOLD (second-level backward finish, etd_unfold2)
    ZYArgs zargs{};                              // ZYFOLD (z unfold + y stack, etd_unfold_fold_zy)
    int th_epi = 0;
    const void* src_fn = nullptr;                // SOURCE / THOMAS kernel
    unsigned src_blocks = 0;
    void* dst = nullptr;                         // COPY2D
    const void* src = nullptr;
    size_t dpitch = 0, spitch = 0, width = 0, height = 0;
    std::vector<Piece> sends, recvs;             // EXCHANGE (matched by order per peer)
    std::string name;
};

struct StageStat {
    std::string name;
    double ms = 0;
    long launches = 0;
    double flops = 0, bytes = 0;
    double dense_flops = 0;
};

// Logical extents + strides of one buffer family (the slab, or the z-stage rows).
struct View {
    int nx = 1, ny = 1, nz = 1;
    long long pitch = 0, plane = 0, F = 0;
    int gj0 = 0, gz0 = 0;
};

static void partition(int n, int G, int r, int& lo, int& hi) {
    const int base = n / G, rem = n % G;
    lo = r * base + std::min(r, rem);
    hi = lo + base + (r < rem ? 1 : 0);
}

// ------------------------------------------------------------ sharded schedule
// Host-only description of the data movement of one sharded step (z-slab
// layout for the x/y stages, y-row layout for the z stage).  Offsets and sizes
// are in elements relative to the named buffers; build_plan turns the records
// into device ops and etd_sharded_schedule exports them for the CPU
// multi-process test (tests/test_dist_cpu.py), which runs the same schedule
// over gloo.
//
// The z stage runs in `C` chunks of each rank's y rows so the exchanges overlap
// the z transforms: the forward exchange of chunk k+1 and the backward
// exchange of chunk k-1 run on the communication stream while chunk k's source
// pass and z transforms run on the compute stream.  Chunk k of rank r owns the
// rows partition(njr, C, k) of its y-row range; its z-stage buffers are a
// separate [field][z][row][x] block (zin/Zz/Wz are the concatenation of the
// chunk blocks), so every exchanged piece lands contiguously.
enum SchedBuf { SB_STATE = 0, SB_SEND = 1, SB_ZIN = 2, SB_WZ = 3, SB_RECV = 4, SB_W = 5 };
enum SchedKind { SK_COPY = 0, SK_SEND = 1, SK_RECV = 2 };
enum SchedPhase { SP_PACK = 0, SP_FWD = 1, SP_BACK = 2, SP_UNPACK = 3 };
struct SchedRec {
    long long kind, phase, peer;
    long long dbuf, doff, dpitch;   // COPY: 2D copy, width/height in elements/rows
    long long sbuf, soff, spitch;   // SEND/RECV: buffer in (sbuf|dbuf), offset, count
    long long width, height, count;
    long long chunk;                // z-stage chunk the record belongs to
};
static constexpr int kZChunks = 4;  // z-stage chunks of a sharded step

// Rows [lo, hi) (relative to rank s's first y row) of chunk k, and the
// element offset of rank r's chunk-k z-stage block (2 ns fields of nz * rows * pitch).
struct ZChunks {
    int G, C;
    std::vector<int> zl, zh, jl, jh;
    long long ns2, pitch, nz;
    void rows(int s, int k, int& lo, int& hi) const { partition(jh[s] - jl[s], C, k, lo, hi); }
    long long nrows(int s, int k) const { int a, b; rows(s, k, a, b); return b - a; }
    long long base(int r, int k) const {
        long long o = 0;
        for (int i = 0; i < k; ++i) o += ns2 * nz * nrows(r, i) * pitch;
        return o;
    }
};
static ZChunks zchunks(int ny, int nz, int ns, int G, long long pitch, int C) {
    ZChunks z{G, C, std::vector<int>(G), std::vector<int>(G), std::vector<int>(G), std::vector<int>(G),
              2LL * ns, pitch, nz};
    for (int s = 0; s < G; ++s) {
        partition(nz, G, s, z.zl[s], z.zh[s]);
        partition(ny, G, s, z.jl[s], z.jh[s]);
    }
    return z;
}

static std::vector<SchedRec> sharded_schedule(int nx, int ny, int nz, int ns, int G, int r, long long pitch,
                                              int C) {
    (void)nx;
    const ZChunks zc = zchunks(ny, nz, ns, G, pitch, C);
    const long long nzr = zc.zh[r] - zc.zl[r];
    const long long plane = pitch * ny, F = plane * nzr;  // slab field
    // send blocks (peer s, chunk k): [c < ns][z in my slab][rows of (s,k)][x]
    // receive blocks (peer s, chunk k): [c < 2 ns][z in my slab][rows of (s,k)][x]
    std::vector<long long> sblock(G * C), rblock(G * C);
    long long so = 0, ro = 0;
    for (int s = 0; s < G; ++s)
        for (int k = 0; k < C; ++k) {
            const long long nk = zc.nrows(s, k);
            sblock[s * C + k] = so;
            so += ns * nzr * nk * pitch;
            rblock[s * C + k] = ro;
            ro += 2 * ns * nzr * nk * pitch;
        }
    std::vector<SchedRec> out;
    auto rec = [&](SchedRec x) { out.push_back(x); };
    // pack: state[c][my z][rows of (s,k)] -> send[(s,k)][c]
    for (int s = 0; s < G; ++s)
        for (int k = 0; k < C; ++k) {
            int a, b;
            zc.rows(s, k, a, b);
            const long long nk = b - a;
            if (nk == 0) continue;
            for (int c = 0; c < ns; ++c)
                rec({SK_COPY, SP_PACK, s, SB_SEND, sblock[s * C + k] + c * nzr * nk * pitch, nk * pitch, SB_STATE,
                     c * F + (zc.jl[s] + a) * pitch, plane, nk * pitch, nzr, nk * pitch * nzr, k});
        }
    for (int k = 0; k < C; ++k) {
        const long long mk = zc.nrows(r, k), planek = pitch * mk, Fk = planek * nz, bk = zc.base(r, k);
        // forward exchange of chunk k: my rows' z planes from every peer
        for (int s = 0; s < G; ++s) {
            const long long nks = zc.nrows(s, k), nzs = zc.zh[s] - zc.zl[s];
            for (int c = 0; c < ns; ++c) {
                if (nks) rec({SK_SEND, SP_FWD, s, 0, 0, 0, SB_SEND, sblock[s * C + k] + c * nzr * nks * pitch, 0, 0, 0,
                              nzr * nks * pitch, k});
                if (mk) rec({SK_RECV, SP_FWD, s, SB_ZIN, bk + c * Fk + zc.zl[s] * planek, 0, 0, 0, 0, 0, 0,
                             nzs * planek, k});
            }
        }
        // backward exchange of chunk k: the 2 ns z-filtered fields back to the slab owners
        for (int c = 0; c < 2 * ns; ++c)
            for (int s = 0; s < G; ++s) {
                const long long nks = zc.nrows(s, k), nzs = zc.zh[s] - zc.zl[s];
                if (mk) rec({SK_SEND, SP_BACK, s, 0, 0, 0, SB_WZ, bk + c * Fk + zc.zl[s] * planek, 0, 0, 0,
                             nzs * planek, k});
                if (nks) rec({SK_RECV, SP_BACK, s, SB_RECV, rblock[s * C + k] + c * nzr * nks * pitch, 0, 0, 0, 0, 0,
                              0, nzr * nks * pitch, k});
            }
    }
    // unpack: recv[(s,k)][c][my z][rows] -> W[c][my z][rows of (s,k)]
    for (int s = 0; s < G; ++s)
        for (int k = 0; k < C; ++k) {
            int a, b;
            zc.rows(s, k, a, b);
            const long long nk = b - a;
            if (nk == 0) continue;
            for (int c = 0; c < 2 * ns; ++c)
                rec({SK_COPY, SP_UNPACK, s, SB_W, c * F + (zc.jl[s] + a) * pitch, plane, SB_RECV,
                     rblock[s * C + k] + c * nzr * nk * pitch, nk * pitch, nk * pitch, nzr, nk * pitch * nzr, k});
        }
    return out;
}

// Where each y row of this rank's slab lands in the receive blocks of the backward
// exchange (sharded_schedule's layout: block (s, k) = [c < 2 ns][my z][rows of (s,k)][x]):
// {element offset, field stride, z stride} per global y row.  The sharded level-2
// y stack pass reads the slab straight from there (no unpack copy).
static std::vector<long long> recv_row_table(int ny, int nz, int ns, int G, int r, long long pitch, int C) {
    const ZChunks zc = zchunks(ny, nz, ns, G, pitch, C);
    const long long nzr = zc.zh[r] - zc.zl[r];
    std::vector<long long> t(3 * (size_t)ny, 0);
    long long ro = 0;
    for (int s = 0; s < G; ++s)
        for (int k = 0; k < C; ++k) {
            int a, b;
            zc.rows(s, k, a, b);
            const long long nk = b - a;
            for (int j = zc.jl[s] + a; j < zc.jl[s] + b; ++j) {
                t[3 * j] = ro + (j - zc.jl[s] - a) * pitch;
                t[3 * j + 1] = nzr * nk * pitch;
                t[3 * j + 2] = nk * pitch;
            }
            ro += 2 * ns * nzr * nk * pitch;
        }
    return t;
}

struct Plan {
    etd_desc d{};
    int dim = 2, ns = 1;
    int G = 1, rank = 0;
    bool sharded = false, local_group = false;
    int nx = 1, ny = 1, nz = 1;      // global interior extents
    int npad[3] = {0, 0, 0};
    long long pitch = 0;
    View slab;                       // x/y-stage (z-slab) view
    std::vector<View> zch;           // sharded: z-stage views of this rank's y-row chunks
    std::vector<long long> zbase;    //   and their offsets in zin / Zz / Wz
    int zC = 1;                      // z-stage chunks
    cudaStream_t xstream = nullptr;  // sharded: exchange stream (high priority)
    std::vector<cudaEvent_t> sev;    // sharded: stream-ordering events
    std::vector<int> zlo, zhi, jlo, jhi;
    double tau = 0;
    cudaStream_t stream = nullptr;
    double* state[2] = {nullptr, nullptr};
    double* Z = nullptr;
    double* W = nullptr;
    double* sendbuf = nullptr;       // sharded: forward-exchange send blocks
    double* zin = nullptr;           // sharded: z-stage input (U,V gathered along z)
    double* Zz = nullptr;
    double* Wz = nullptr;
    double* recvb = nullptr;         // sharded: backward-exchange receive blocks
    int* codes = nullptr;            // sharded: [G] gathered fail codes; codes[G] = own
    double* PR[3] = {nullptr, nullptr, nullptr};
    double* PTR[3] = {nullptr, nullptr, nullptr};
    // parity split (etd_kernels.cuh, FOLD): per axis h and the interleaved h-column
    // matrices of the forward (FF) and backward (FB) half transforms, stored in the
    // axis' B layout (x: [2h][ldx] rows; y/z: [h][2h], output index contiguous)
    bool fold[3] = {false, false, false};
    int fh[3] = {0, 0, 0};
    double* FF[3] = {nullptr, nullptr, nullptr};
    double* FB[3] = {nullptr, nullptr, nullptr};
    // second-level split: forward = etd_fold2 stack + FOLD 5 (GA, even
    // modes) + FOLD 4 (GB, odd modes); FB then reads the level-2 mode positions
    bool fold2[3] = {false, false, false};
    bool fold2_all = false;          // every axis split twice: the step runs the level-2 schedule
    double* GA[3] = {nullptr, nullptr, nullptr};
    double* GB[3] = {nullptr, nullptr, nullptr};
    double* GO[3] = {nullptr, nullptr, nullptr};     // level-2 backward: FOLD 4 over (sigma, delta)
    double* GE[3] = {nullptr, nullptr, nullptr};     //   and FOLD 2 over the odd-mode group
    double* G6[3] = {nullptr, nullptr, nullptr};     // fused level-2 backward (etd_back6, back6_matrix)
    bool back6 = false;                              // the level-2 backward runs fused (ETD_BACK6=0: r01 path)
    double* dvec = nullptr;          // [order 3][axis][slot 9][species 2][dmax]; order 1 = parity-major, 2 = level 2
    double* sintab[3] = {nullptr, nullptr, nullptr};  // sin(pi * coord) per axis (global extents)
    int dmax = 0;
    StepStatus* status = nullptr;
    StepStatus* status_host = nullptr;
    mutable unsigned long long* trace = nullptr;  // ETD_CTA_TRACE=<stage name part>: CTA phase clocks (diagnostic)
    int cur = 0;
    std::vector<Op> steps[2];
    cudaGraphExec_t graph[2] = {nullptr, nullptr};
    bool profiling = false;
    std::vector<StageStat> stats;
    void* comm = nullptr;            // ncclComm_t
    cudaStream_t cstream = nullptr;  // host<->device copy stream of the pipelined advance
    std::vector<cudaEvent_t> xev;    // its chunk events
    int state_fields = 0;            // fields per state buffer (ns on the level-2 schedule, else 2 ns)
    long long* recv_rows = nullptr;  // sharded level 2: per slab y row, {offset, field stride, z stride} in recvb
    double* mirror = nullptr;        // pinned host mirror of the state (pageable etd_advance buffers)
    size_t mirror_elems = 0;
    // BackendKind::Thomas: per-axis factors [species][pole][mul, piv, 1/piv][n],
    // per-axis launch templates, forward-sweep scratch and pole partial sums
    bool thomas = false;
    double2* thfac[3] = {nullptr, nullptr, nullptr};
    ThomasArgs thbase[3] = {};
    double2* thscr = nullptr;
    long long th_cap = 0;            // thscr capacity in double2
    long long th_need = 0;           // largest checkpoint scratch of the built passes
    int nsm = 148;
    long long th_T = 0;

    ~Plan() {
        for (auto& g : graph)
            if (g) cudaGraphExecDestroy(g);
        for (double* p : {state[0], state[1], Z, W, dvec, sendbuf, zin, Zz, Wz, recvb}) if (p) cudaFree(p);
        if (codes) cudaFree(codes);
        if (recv_rows) cudaFree(recv_rows);
        for (double* t : sintab) if (t) cudaFree(t);
        for (double2* t : thfac) if (t) cudaFree(t);
        if (thscr) cudaFree(thscr);
        for (int a = 0; a < 3; ++a)
            for (double* m : {PR[a], PTR[a], FF[a], FB[a], GA[a], GB[a], GO[a], GE[a], G6[a]}) if (m) cudaFree(m);
        if (trace) {
            // dump {count, records of smid, block, t0..t3} for tools/cta_trace.py
            std::vector<unsigned long long> h(8 + 8192 * 24);
            if (cudaMemcpy(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost) == cudaSuccess) {
                const char* path = std::getenv("ETD_CTA_TRACE_OUT");
                if (FILE* f = std::fopen(path ? path : "cta_trace.bin", "wb")) {
                    std::fwrite(h.data(), 8, h.size(), f);
                    std::fclose(f);
                }
            }
            cudaFree(trace);
        }
        if (status) cudaFree(status);
        if (status_host) cudaFreeHost(status_host);
        if (mirror) cudaFreeHost(mirror);
        if (comm) Nccl::get().CommDestroy(comm);
        for (auto e : xev) cudaEventDestroy(e);
        for (auto e : sev) cudaEventDestroy(e);
        if (xstream) cudaStreamDestroy(xstream);
        if (cstream) cudaStreamDestroy(cstream);
        if (stream) cudaStreamDestroy(stream);
    }

    // d-vector slot of an axis in natural mode order, or parity-major on folded axes
    const double* dv(int axis, int slot) const { return dvn(axis, slot, fold[axis] ? (fold2[axis] ? 2 : 1) : 0); }
    const double* dvn(int axis, int slot, int order) const {
        return dvec + (((size_t)3 * order + axis) * 9 + slot) * 2 * dmax;
    }
    static int n_axis(const View& v, int a) { return a == 0 ? v.nx : a == 1 ? v.ny : v.nz; }

    // ---- maps over stacked fields (one TMA box per stage per operand set) ----
    // MODE 0 view: dims {nx, R, count}, box {16, BM, count} -> smem [op][BM][16]
    static CUtensorMap mapA_x(const View& v, const double* base, int count, int bm, long long fs = 0) {
        const unsigned long long dims[3] = {(unsigned long long)v.nx, (unsigned long long)v.ny * v.nz,
                                            (unsigned long long)count};
        const unsigned long long st[2] = {(unsigned long long)v.pitch, (unsigned long long)(fs ? fs : v.F)};
        const unsigned box[3] = {16, (unsigned)bm, (unsigned)count};
        return make_map(base, 3, dims, st, box);
    }
    // MODE 1 view: dims {x%16, k, x/16, outer, count}, box {16, 16, BM/16, 1, count}
    // -> smem [op][pb][k][16].  x columns past nx read the zero pad of the pitch.
    static CUtensorMap mapA_yz(const View& v, const double* base, int count, bool zaxis, int bm, long long fs = 0) {
        const unsigned long long nk = zaxis ? v.nz : v.ny, no = zaxis ? v.ny : v.nz;
        const unsigned long long sk = zaxis ? v.plane : v.pitch, so = zaxis ? v.pitch : v.plane;
        const unsigned long long dims[5] = {16, nk, (unsigned long long)((v.nx + 15) / 16), no,
                                            (unsigned long long)count};
        const unsigned long long st[4] = {sk, 16, so, (unsigned long long)(fs ? fs : v.F)};
        const unsigned box[5] = {16, 16, (unsigned)(bm / 16), 1, (unsigned)count};
        return make_map(base, 5, dims, st, box);
    }
    // B: row-major n x n (zero-padded to npad).  MODE 0: dims {k, n} box {16, BN};
    // MODE 1: dims {n%16, k, n/16} box {16, 16, BN/16} -> smem [nb][k][16]
    CUtensorMap mapB(const double* M, int axis, int mode, int bn) const {
        const int n = d.n[axis];
        if (mode == 0) {
            const unsigned long long dims[2] = {(unsigned long long)n, (unsigned long long)n};
            const unsigned long long st[1] = {(unsigned long long)npad[axis]};
            const unsigned box[2] = {16, (unsigned)bn};
            return make_map(M, 2, dims, st, box);
        }
        const unsigned long long dims[3] = {16, (unsigned long long)n, (unsigned long long)(npad[axis] / 16)};
        const unsigned long long st[2] = {(unsigned long long)npad[axis], 16};
        const unsigned box[3] = {16, 16, (unsigned)(bn / 16)};
        return make_map(M, 3, dims, st, box);
    }
    // parity-split B: 2h interleaved rows x h columns (fold_matrices layout; GA/GB with h = H)
    CUtensorMap mapB_fold(const double* M, int axis, int mode, int bn, int hh = 0) const {
        const unsigned long long h = hh ? hh : fh[axis];
        if (mode == 0) {
            const unsigned long long dims[2] = {h, 2 * h};
            const unsigned long long st[1] = {(unsigned long long)round16(h)};
            const unsigned box[2] = {16, (unsigned)bn};
            return make_map(M, 2, dims, st, box);
        }
        const unsigned long long dims[3] = {16, h, 2 * h / 16};
        const unsigned long long st[2] = {2 * h, 16};
        const unsigned box[3] = {16, 16, (unsigned)(bn / 16)};
        return make_map(M, 3, dims, st, box);
    }
    static unsigned long long round16(unsigned long long x) { return (x + 15) / 16 * 16; }
    // fused level-2 backward B (back6_matrix): 4H rows x H columns; mode 0 rows
    // contiguous (leading dimension round16(H)), mode 1 the transpose [H][4H]
    CUtensorMap mapB_back6(const double* M, int axis, int mode, int bn) const {
        const unsigned long long H = fh[axis] / 2, R = (4 * H + 63) / 64 * 64;
        if (mode == 0) {
            const unsigned long long dims[2] = {H, R};
            const unsigned long long st[1] = {round16(H)};
            const unsigned box[2] = {16, (unsigned)bn};
            return make_map(M, 2, dims, st, box);
        }
        const unsigned long long dims[3] = {16, H, R / 16};
        const unsigned long long st[2] = {R, 16};
        const unsigned box[3] = {16, 16, (unsigned)(bn / 16)};
        return make_map(M, 3, dims, st, box);
    }

    ContractArgs base_args(const View& v, int axis) const {
        ContractArgs a{};
        a.n_axis = n_axis(v, axis);
        a.kext = a.n_axis;
        a.m_extent = axis == 0 ? v.ny * v.nz : v.nx;
        a.zaxis = axis == 2;
        a.nspecies = ns;
        a.pitch = v.pitch;
        a.plane = v.plane;
        a.out_stride = v.F;
        a.aux_stride = v.F;
        a.dstride = dmax;
        a.src_kind = d.src_kind;
        for (int i = 0; i < 8; ++i) a.sp[i] = d.src_params[i];
        a.ny_local = v.ny;
        a.gj0 = v.gj0;
        a.gz0 = v.gz0;
        a.status = status;
        a.tau = tau;
        a.commit = sharded ? 0 : 1;
        a.mix_w2 = 1;
        a.sinx = sintab[0];
        a.siny = sintab[1];
        a.sinz = dim == 3 ? sintab[2] : nullptr;
        return a;
    }

    // The per-step source pass f(t, U(,V)) into the f slots of the stack at `buf`,
    // or (fold_axis 1/2) the whole stack folded along that axis into `fold_out`.
    Op source_op(const View& v, double* buf, double* fold_out = nullptr, int fold_axis = 0, bool fold2 = false) const {
        Op o;
        o.kind = Op::SOURCE;
        o.name = "source";
        o.L.name = "source";
        SourceArgs& a = o.sargs;
        a.fold = 0;
        a.fh = 0;
        a.fold_out = nullptr;
        a.x0 = 0;
        a.x1 = v.nx;
        a.buf = buf;
        a.F = v.F;
        a.pitch = v.pitch;
        a.plane = v.plane;
        a.nx = v.nx;
        a.ny = v.ny;
        a.nz = v.nz;
        a.j0 = 0;
        a.j1 = v.ny;
        a.gj0 = v.gj0;
        a.gz0 = v.gz0;
        a.nspecies = ns;
        for (int i = 0; i < 8; ++i) a.sp[i] = d.src_params[i];
        a.sinx = sintab[0];
        a.siny = sintab[1];
        a.sinz = dim == 3 ? sintab[2] : nullptr;
        a.status = status;
        o.src_fn = pick_source(d.src_kind, ns, fold_axis && fold2);
        o.src_blocks = (unsigned)std::min<long long>((long long)v.ny * v.nz, 148LL * 16);
        const double pts = (double)v.nx * v.ny * v.nz;
        o.L.flops = 0.0;
        o.L.bytes = pts * 8.0 * 2 * ns;  // read U(,V), write fU(,fV)
        if (fold_axis) {
            a.fold = fold_axis;
            a.fh = fh[fold_axis];
            a.fold_out = fold_out;
            a.fold2 = fold2 ? 1 : 0;
            o.L.bytes = pts * 8.0 * 3 * ns;  // read U(,V), write the folded [U,(V),fU,(fV)]
        }
        return o;
    }

    // The second-level split stack (etd_fold2) of `nf` fields along `axis`: in -> out
    // (stacks with field stride v.F); from1: `in` holds the first-level stack.
    Op fold_op(const View& v, const std::string& name, int axis, const double* in, double* out, int nf,
               bool from1 = false) const {
        Op o;
        o.kind = Op::FOLD;
        o.name = name;
        o.L.name = name;
        o.L.mode = axis == 0 ? 0 : 1;
        Fold2Args& a = o.fargs;
        a.in = in;
        a.out = out;
        a.Fin = a.Fout = v.F;
        a.nf = nf;
        a.axis = axis;
        a.n = n_axis(v, axis);
        a.H = fh[axis] / 2;
        a.from1 = from1 ? 1 : 0;
        a.pitch = v.pitch;
        a.plane = v.plane;
        a.nx = v.nx;
        a.ny = v.ny;
        a.nz = v.nz;
        a.x0 = 0;
        a.x1 = v.nx;
        a.r0 = 0;
        a.r1 = (long long)v.ny * v.nz;
        a.rows = nullptr;
        {
            const char* e = getenv("ETD_FOLDX4");  // A/B: 0 = one orbit per thread, 8-byte accesses
            a.x4 = (axis == 0 && !from1 && a.H % 4 == 0 && !(e && atoi(e) == 0)) ? 1 : 0;
        }
        const double pts = (double)v.nx * v.ny * v.nz;
        o.L.flops = 0.0;
        o.L.bytes = pts * 8.0 * 2 * nf;
        o.src_blocks = 148u * 16u;
        return o;
    }

    // The second-level backward's finishing pass (etd_unfold2) of the intermediate
    // stack `in` along `axis`, with the stage epilogue `uf` fused (UF_WHAT_SRC: What
    // -> out, f's level-2 stack -> fout; UF_UPDATE: aux + g -> out, commit).
    Op unfold_op(const View& v, const std::string& name, int axis, int uf, const double* in, double* out, int nf,
                 const double* aux = nullptr, double* fout = nullptr) const {
        Op o;
        o.kind = Op::UNFOLD;
        o.name = name;
        o.L.name = name;
        o.L.mode = axis == 0 ? 0 : 1;
        o.L.epi = uf == UF_UPDATE ? EPI_UPDATE : uf == UF_WHAT_SRC ? EPI_WHAT_SRC : EPI_STORE;
        o.L.args.out = out;  // the pipelined advance downloads U' from here
        Unfold2Args& a = o.uargs;
        a.in = in;
        a.out = out;
        a.Fin = a.Fout = a.Faux = v.F;
        a.nf = nf;
        a.axis = axis;
        a.n = n_axis(v, axis);
        a.H = fh[axis] / 2;
        a.pitch = v.pitch;
        a.plane = v.plane;
        a.nx = v.nx;
        a.ny = v.ny;
        a.nz = v.nz;
        a.x0 = 0;
        a.x1 = v.nx;
        a.r0 = 0;
        a.r1 = (long long)v.ny * v.nz;
        a.aux = aux;
        a.fout = fout;
        a.status = status;
        a.tau = tau;
        a.commit = (uf == UF_UPDATE && !sharded) ? 1 : 0;
        for (int i = 0; i < 8; ++i) a.sp[i] = d.src_params[i];
        a.sinx = sintab[0];
        a.siny = sintab[1];
        a.sinz = dim == 3 ? sintab[2] : nullptr;
        a.ny_local = v.ny;
        a.gj0 = v.gj0;
        a.gz0 = v.gz0;
        o.src_fn = pick_unfold(uf == UF_WHAT_SRC ? d.src_kind : 0, uf);
        o.src_blocks = 148u * 16u;
        const double pts = (double)v.nx * v.ny * v.nz;
        o.L.flops = 0.0;
        o.L.bytes = pts * 8.0 * nf * (uf == UF_STORE ? 2 : (uf == UF_WHAT_SRC && aux) ? 4 : 3);
        return o;
    }

    // A transform along `axis` of `S` stacked operands at `in` (L loaded), M = P^T (fwd) or P.
    // Folded axes run the parity-split kernels unless `dense` (the dense n x n
    // contraction; kernel-level tests of a single direction use it).
    // x forward transforms fold as FOLD 3 (mirror from the x-reversed operand
    // `in_rev`) or FOLD 4 (`in` pre-folded); y/z forward as FOLD 1; backward FOLD 2.
    // part 1 / 2: the even- / odd-mode launch of a second-level split forward
    // transform (FOLD 5 / FOLD 4) of the etd_fold2 stack at `in`.
    Launch transform(const View& v, const std::string& name, int axis, bool back, int S, int epi, bool pro,
                     const double* in, double* out, bool dense = false, const double* in_rev = nullptr,
                     bool prefolded = false, int part = 0, long long fstride = 0) const {
        Launch L;
        int fold = (this->fold[axis] && !dense && !pro) ? (back ? 2 : 1) : 0;
        if (fold == 1 && prefolded) fold = 4;
        if (part) {
            if (!fold2[axis] || back != (part >= 3) || pro || dense)
                throw ConfigError("second-level split launch on an ineligible axis / direction");
            fold = part == 1 ? 5 : part == 2 ? 4 : part == 3 ? 4 : part == 6 ? 6 : 2;
        } else if (fold == 1 && axis == 0) {
            if (epi == EPI_CORR) fold = 4;
            else if (in_rev) fold = 3;
            else throw ConfigError("x forward parity split needs the x-reversed operand");
        }
        L.name = name;
        const int mode = axis == 0 ? 0 : 1;
        L.mode = mode;
        L.S = S;
        L.epi = epi;
        L.pro = pro;
        const int nax = n_axis(v, axis);
        const long long mext = axis == 0 ? (long long)v.ny * v.nz : v.nx;
        const unsigned gz = mode == 0 ? 1u : (axis == 1 ? (unsigned)v.nz : (unsigned)v.ny);
        // Tile class (measured per stage on configs 0-4, tools/tile_sweep.py):
        //  * short contractions (n <= 255): 32x32 tiles (T=2) — pipeline fill and
        //    drain dominate larger tiles at 16 k-tiles
        //  * otherwise 2 CTAs/SM with 32 accumulators (T=3) when that fills two waves
        //  * else the 8-warp tile (T=0) when it fills two waves, else T=2
        const int H2 = fh[axis] / 2;
        const int nrows = part == 6 ? (4 * H2 + 63) / 64 * 64 : part ? 2 * H2 : fold ? 2 * fh[axis] : nax;  // B rows
        const int kext = part ? H2 : fold ? fh[axis] : nax;
        auto ctas = [&](int t) {
            const KernelSpec k = pick(mode, S, epi, pro, d.src_kind, t, fold);
            return (long long)((nrows + k.bn - 1) / k.bn) * ((mext + k.bm - 1) / k.bm) * gz;
        };
        int tile;
        if (fold == 6) {
            // fused level-2 backward: 2 CTAs/SM with a 2-deep ring when that fills two
            // waves, else the 1-CTA/SM 4-stage class, else the small tile
            tile = ctas(3) >= 2 * 148 ? 3 : ctas(0) >= 148 ? 0 : 2;
        } else if (fold) {
            // parity-split kernels (tools/tile_sweep.py on configs 1-4, profiles/r01_tile_sweep_fold.txt):
            //  * S = 4 has one class (32x128, 8 warps)
            //  * 2 CTAs/SM when that fills two waves, except the S = 2 update (T=3 spills)
            //  * else the 8-warp tile down to ~2/3 of a wave (2D n = 1023 y stages), else 32x32
            // (the FOLD 5 sigma/delta epilogue spills under the 2-CTA/SM register cap)
            if (S == 4) tile = 0;
            else if (ctas(3) >= 2 * 148 && !(epi == EPI_UPDATE && S == 2) && !(part == 1 && S == 2 && epi == EPI_CORR))
                tile = 3;
            else if (ctas(0) >= 100) tile = 0;
            else tile = 2;
        } else if (kext <= 255) tile = 2;
        else if (ctas(3) >= 2 * 148) tile = 3;
        else if (ctas(0) >= 2 * 148) tile = 0;
        else tile = 2;
        if (const char* f = std::getenv("ETD_FORCE_TILE"))  // tests: exercise every tile class
            if (f[0] >= '0' && f[0] <= '3' && f[1] == 0) tile = f[0] - '0';
        if (fold == 6)
            if (const char* f = std::getenv(mode == 0 ? "ETD_BACK6_TILE_X" : "ETD_BACK6_TILE_YZ"))  // A/B
                if (f[0] >= '0' && f[0] <= '3' && f[1] == 0) tile = f[0] - '0';
        if (fold == 6 && tile == 1) tile = 0;  // the fused backward has no 4-warp 64x64 class
        L.tile = tile;
        L.fold = fold;
        L.k = pick(mode, S, epi, pro, d.src_kind, tile, fold);
        const int loaded = pro ? S / 2 : S;
        L.tmA = mode == 0 ? mapA_x(v, in, loaded, L.k.bm, fstride) : mapA_yz(v, in, loaded, axis == 2, L.k.bm, fstride);
        L.tmA2 = fold == 3 ? mapA_x(v, in_rev, loaded, L.k.bm) : L.tmA;
        if (part == 6) {
            L.tmB = mapB_back6(G6[axis], axis, mode, L.k.bn);
        } else if (part) {
            const double* M = part == 1 ? GA[axis] : part == 2 ? GB[axis] : part == 3 ? GO[axis] : GE[axis];
            L.tmB = mapB_fold(M, axis, mode, L.k.bn, H2);
        } else if (fold) {
            L.tmB = mapB_fold(back ? FB[axis] : FF[axis], axis, mode, L.k.bn);
        } else {
            // fwd (M = P^T): mode 0 needs row-major P^T, mode 1 row-major P; back swaps
            const double* M = (mode == 0) != back ? PTR[axis] : PR[axis];
            L.tmB = mapB(M, axis, mode, L.k.bn);
        }
        L.args = base_args(v, axis);
        L.args.out = out;
        if (fstride) L.args.out_stride = fstride;
        L.args.kext = kext;
        L.args.fold_h = fh[axis];
        if (part == 1) {
            L.args.n_axis = 2 * H2;  // the FOLD 2 mirror pairs (q, h-1-q) of the even-mode group
            L.args.fold_h = H2;
            L.args.sd_out = 1;       // the level-2 backward reads (sigma, delta)
        } else if (part == 2) {
            L.args.fold_h = H2;
            L.args.kbase = 2 * H2;
            L.args.nbase = 2 * H2;
        } else if (part == 3) {
            L.args.n_axis = 2 * H2;  // o at even i -> [0, H), odd i -> [H, 2H) of the intermediate stack
            L.args.fold_h = H2;
        } else if (part == 4) {
            L.args.n_axis = 2 * H2 - 1;  // the DST-I of size h - 1: e_i and e_{2H-2-i} -> [2H, 4H - 1)
            L.args.fold_h = H2;
            L.args.kbase = 2 * H2;
            L.args.nbase = 2 * H2;
        } else if (part == 6) {
            L.args.fold_h = H2;          // the whole level-2 backward in one launch (etd_back6)
        }
        const unsigned gx = (nrows + L.k.bn - 1) / L.k.bn;
        const unsigned gy = (unsigned)((mext + L.k.bm - 1) / L.k.bm);
        L.grid = dim3(gx, gy, gz);
        if (const char* e = std::getenv("ETD_CTA_TRACE"))
            if (fold == 6 && name.find(e) != std::string::npos) {
                if (!trace) {
                    ETD_CK(cudaMalloc(&trace, (8 + 8192 * 24) * 8));
                    ETD_CK(cudaMemset(trace, 0, (8 + 8192 * 24) * 8));
                }
                L.args.trace = trace;
            }
        const double pts = (double)v.nx * v.ny * v.nz;
        // executed (= algorithmic) FLOPs of this launch: 2 n per point dense,
        // 2 (2h) h / n per point split (half)
        L.flops = 2.0 * ((double)nrows * kext / nax) * pts * S;
        L.dense_flops = 2.0 * nax * pts * S * ((part && part != 6) ? 0.5 : 1.0);
        int outs = S, aux = 0;
        if (epi == EPI_WHAT_SRC) outs = 2 * S;
        if (epi == EPI_CORR || epi == EPI_UPDATE) aux = S;
        if (part == 6 && epi == EPI_WHAT_SRC) aux = S;  // w2 in physical space
        L.bytes = pts * 8.0 * (loaded + outs + aux) * ((part && part != 6) ? 0.5 : 1.0);
        return L;
    }

    // One Thomas pass along `axis` (apply_Q_thomas, thomas.cpp:128-160, with the
    // stage epilogue `epi`) over the operand stack `stack` (2 ns fields, stride F):
    //   TH_STORE   Q_ell of fields [f0, f0 + nfields) -> out (same field index)
    //   TH_WHAT    (x) the predictor + f(t + tau) of every species: W stack -> out
    //   TH_UPDATE  (x) the corrector U1 = What + tau Q3(fw): fw at stack[fin_off + c],
    //              What at stack[c] -> out[c], c < nfields; commits the step
    // Scratch (checkpoints) is sized after the schedule is built (th_need).
    Op thomas_op(const std::string& name, int axis, int epi, const double* stack, double* out, int nfields,
                 int ell, int f0 = 0, int fin_off = 0) {
        const View& v = slab;
        const int mode = axis == 0 ? 0 : 1;
        Op o;
        o.kind = Op::THOMAS;
        o.name = name;
        o.L.name = name;
        o.L.mode = mode;
        o.th_epi = epi;
        ThomasArgs a = thbase[axis];
        a.out = out;
        a.ell = ell;
        a.f_first = f0;
        a.fin_off = fin_off;
        a.commit = epi == TH_UPDATE;
        a.aux = stack;
        const int nfl = epi == TH_WHAT ? 1 : nfields;
        const unsigned long long nst = 2ull * ns;
        const ThomasSpec k = pick_thomas(mode, epi, ns, d.src_kind, a.npoles);
        const int PP = k.pencils;
        if (mode == 1) {
            const bool z = axis == 2;
            a.es = z ? v.plane : v.pitch;
            a.so = z ? v.pitch : v.plane;
            a.npen = v.nx;
            a.nouter = z ? v.ny : v.nz;
            a.ptiles = (v.nx + PP - 1) / PP;
            // {x%16, axis, x/16, outer, field}, box {16, 16, 8, 1, 1} -> [x-block][16][16]
            const unsigned long long dims[5] = {16, (unsigned long long)a.n, (unsigned long long)((v.nx + 15) / 16),
                                                (unsigned long long)a.nouter, nst};
            const unsigned long long st[4] = {(unsigned long long)a.es, 16, (unsigned long long)a.so,
                                              (unsigned long long)v.F};
            const unsigned box[5] = {16, 16, (unsigned)(PP / 16), 1, 1};
            o.L.tmA = make_map(stack, 5, dims, st, box);
        } else {
            a.pitch = v.pitch;
            a.npen = v.ny * v.nz;
            a.nouter = 1;
            a.ptiles = (a.npen + PP - 1) / PP;
            // {x, row, field}, box {16, pencils, 1}, 128B swizzle -> [row][16]
            const unsigned long long dims[3] = {(unsigned long long)v.nx, (unsigned long long)a.npen, nst};
            const unsigned long long st[2] = {(unsigned long long)v.pitch, (unsigned long long)v.F};
            const unsigned box[3] = {16, (unsigned)PP, 1};
            o.L.tmA = make_map(stack, 3, dims, st, box);
        }
        a.ntiles = (long long)a.ptiles * a.nouter * nfl;
        const long long G = std::max<long long>(1, std::min<long long>(a.ntiles, (long long)nsm * k.occ));
        // checkpoints per thread: rhs per thread x poles x chunks (128 threads per CTA)
        const long long R = (epi == TH_WHAT && ns == 2) ? 2 : thomas_rhs(epi, ns), K = thomas_chunk((int)R);
        th_need = std::max(th_need, R * a.npoles * ((a.n + K - 1) / K) * G * 128);
        o.targs = a;
        o.src_fn = k.fn;
        o.src_blocks = (unsigned)G;
        o.L.k.smem = k.smem;
        const double pts = (double)v.nx * v.ny * v.nz;
        const int rhs = epi == TH_WHAT ? 2 * ns : nfields;
        const int outs = epi == TH_WHAT ? 2 * ns : nfields;
        // per pole: forward (mul w, 6 flops) + back (e w, 1/piv w, 2 Re(r w): ~16 flops)
        o.L.flops = pts * rhs * a.npoles * 22.0;
        // algorithmic bytes: operands in, results out (TH_UPDATE also reads What)
        o.L.bytes = pts * 8.0 * (rhs + outs + (epi == TH_UPDATE ? nfields : 0));
        return o;
    }
};

// ------------------------------------------------------------ setup
static int round_up(int x, int m) { return (x + m - 1) / m * m; }

static void check_source(int nspecies, int k) {
    const bool scalar_src = k == ETD_SRC_ZERO || k == ETD_SRC_AC_CUBIC || k == ETD_SRC_POLY3 || k == ETD_SRC_NAN ||
                            k == ETD_SRC_AC_MANUFACTURED || k == ETD_SRC_SINGULAR;
    const bool pair_src = k == ETD_SRC_FHN_CUBIC || k == ETD_SRC_FHN_CLASSIC || k == ETD_SRC_MIRROR_AC ||
                          k == ETD_SRC_DECOUPLED || k == ETD_SRC_ZERO;
    if (nspecies == 2 ? !pair_src : !scalar_src)
        throw ConfigError("the CUDA backend needs a device source descriptor matching the plan (no CPU fallback)");
}

static void drop_graphs(Plan& p) {
    for (auto& g : p.graph)
        if (g) {
            cudaGraphExecDestroy(g);
            g = nullptr;
        }
}

static void set_source(Plan& p, int kind, const double* params) {
    check_source(p.ns, kind);
    p.d.src_kind = kind;
    for (int i = 0; i < 8; ++i) p.d.src_params[i] = params ? params[i] : 0.0;
    for (int par = 0; par < 2; ++par)
        for (auto& op : p.steps[par])
            if (op.kind == Op::SOURCE) {
                for (int i = 0; i < 8; ++i) op.sargs.sp[i] = p.d.src_params[i];
                op.src_fn = pick_source(kind, p.ns, op.sargs.fold && op.sargs.fold2);
            } else if (op.kind == Op::THOMAS) {
                for (int i = 0; i < 8; ++i) op.targs.sp[i] = p.d.src_params[i];
                op.src_fn = pick_thomas(op.L.mode, op.th_epi, p.ns, kind, op.targs.npoles).fn;
            } else if (op.kind == Op::KERNEL) {
                op.L.args.src_kind = kind;
                for (int i = 0; i < 8; ++i) op.L.args.sp[i] = p.d.src_params[i];
                op.L.k = pick(op.L.mode, op.L.S, op.L.epi, op.L.pro, kind, op.L.tile, op.L.fold);
            } else if (op.kind == Op::UNFOLD) {
                for (int i = 0; i < 8; ++i) op.uargs.sp[i] = p.d.src_params[i];
                const int uf = op.L.epi == EPI_WHAT_SRC ? UF_WHAT_SRC : op.L.epi == EPI_UPDATE ? UF_UPDATE : UF_STORE;
                op.src_fn = pick_unfold(uf == UF_WHAT_SRC ? kind : 0, uf);
            }
    drop_graphs(p);
}

static Op kernel_op(Launch L) {
    Op o;
    o.kind = Op::KERNEL;
    o.name = L.name;
    o.L = std::move(L);
    return o;
}

static Op copy_op(const std::string& name, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                  size_t height) {
    Op o;
    o.kind = Op::COPY2D;
    o.name = name;
    o.dst = dst;
    o.dpitch = dpitch;
    o.src = src;
    o.spitch = spitch;
    o.width = width;
    o.height = height;
    return o;
}

static void validate(const etd_desc& d) {
    if (d.dim != 2 && d.dim != 3) throw ConfigError("grid dimension must be 2 or 3");
    if (!(d.tau > 0.0)) throw ConfigError("tau must be positive");
    if (d.nspecies != 1 && d.nspecies != 2) throw ConfigError("nspecies must be 1 or 2");
    if (d.family != ETD_P02 && d.family != ETD_P04 && d.family != ETD_EXACT)
        throw ConfigError("unknown Pade family / backend");
    if (d.backend != ETD_SPECTRAL && d.backend != ETD_THOMAS) throw ConfigError("unknown backend");
    if (d.backend == ETD_THOMAS && d.family == ETD_EXACT)
        throw ConfigError("the exact-exponential reference runs on the spectral backend");
    if (d.backend == ETD_THOMAS && d.world_size > 1)
        throw ConfigError("the Thomas backend runs on one GPU (no z-slab sharding)");
    check_source(d.nspecies, d.src_kind);
    for (int a = 0; a < d.dim; ++a) {
        if (d.n[a] < 1) throw ConfigError("need at least 2 subintervals for a nonempty interior");
        if (!(d.high[a] > d.low[a])) throw ConfigError("upper bound must exceed lower");
    }
    if (!(d.kappa[0] > 0.0) || (d.nspecies == 2 && !(d.kappa[1] > 0.0)))
        throw ConfigError(d.nspecies == 2 ? "component diffusivities must be positive" : "diffusivity must be positive");
    if (d.q < 0.0) throw ConfigError("linear reaction coefficient must be nonnegative");
    const int G = d.world_size < 1 ? 1 : d.world_size;
    if (G > 1) {
        if (d.dim != 3) throw ConfigError("z-slab sharding needs a 3D grid (2D configs run as replicas)");
        if (d.rank < 0 || d.rank >= G) throw ConfigError("rank out of range");
        if (G > d.n[2] || G > d.n[1]) throw ConfigError("more ranks than z planes / y rows");
    }
}

// (Re)allocate the Thomas checkpoint scratch to hold `need` entries and point
// every Thomas op of the step schedule at it.
static void ensure_thomas_scratch(Plan& p, long long need) {
    if (need > p.th_cap) {
        if (p.thscr) ETD_CK(cudaFree(p.thscr));
        p.thscr = nullptr;
        ETD_CK(cudaMalloc(&p.thscr, (size_t)need * sizeof(double2)));
        p.th_cap = need;
        drop_graphs(p);
    }
    for (auto& steps : p.steps)
        for (auto& op : steps)
            if (op.kind == Op::THOMAS) op.targs.scratch = p.thscr;
}

// Parity-split half matrices of one axis (etd_kernels.cuh, FOLD) from the
// reference eigenvector matrix Pc (column-major, P(i,k) = Pc[k n + i],
// operators.cpp:43-53).  h = (n+1)/2; row r of the 2h interleaved rows is
// (block b = r/16, t = r%16): group t/8 (0: even modes, 1: odd modes), index
// q = 8b + t%8.
//   forward  FF[r][c] = P(c, k), k = 2q + group  (the output mode), c < h the folded
//            input index; for odd n the centre column c = h-1 is halved in the even
//            group (s counts it twice) and zero in the odd group (d is 0 there)
//   backward FB[r][c] = P(q, k), k = 2c + group  (the input mode), q the output
//            index; the centre row of the odd group is exactly 0 so that the centre
//            output is o + 0 = o - 0
// Entries with k >= n are 0.  mode 0 (x) stores [2h][round16(h)] (row r
// contiguous); mode 1 (y/z) stores the transpose [h][2h].
static void fold_matrices(const std::vector<double>& Pc, int n, int mode, std::vector<double>& ff,
                          std::vector<double>& fb) {
    const int h = (n + 1) / 2;
    const bool odd = n & 1;
    const int ld = mode == 0 ? (h + 15) / 16 * 16 : 2 * h;
    ff.assign(mode == 0 ? (size_t)2 * h * ld : (size_t)h * ld, 0.0);
    fb.assign(ff.size(), 0.0);
    auto P = [&](int i, int k) { return Pc[(size_t)k * n + i]; };
    auto at = [&](std::vector<double>& m, int r, int c) -> double& {
        return mode == 0 ? m[(size_t)r * ld + c] : m[(size_t)c * ld + r];
    };
    for (int r = 0; r < 2 * h; ++r) {
        const int grp = (r >> 3) & 1, q = (r >> 4) * 8 + (r & 7);
        if (q >= h) continue;
        for (int c = 0; c < h; ++c) {
            const int kf = 2 * q + grp;
            if (kf < n) {
                double v = P(c, kf);
                if (odd && c == h - 1) v = grp == 0 ? 0.5 * v : 0.0;
                at(ff, r, c) = v;
            }
            const int kb = 2 * c + grp;
            if (kb < n) at(fb, r, c) = (odd && q == h - 1 && grp == 1) ? 0.0 : P(q, kb);
        }
    }
}

// Second-level split of an axis with n = 4H - 1, h = 2H.  Mode
// positions: p < h -> mode 2p; h + c -> mode 4c + 1 (c < H), 4(c - H) + 3 (c >= H).
static int fold2_mode(int pos, int n) {
    const int h = (n + 1) / 2, H = h / 2;
    if (pos < h) return 2 * pos;
    const int c = pos - h;
    return c < H ? 4 * c + 1 : 4 * (c - H) + 3;
}
// GA (FOLD 5, even modes): row r = (block b = r/16, t = r%16): group t/8 = parity of
//    the input index i = 2c + group, output q = 8b + t%8 < H; GA[r][c] = P(i, 2q),
//    the centre i = h-1 (odd group, c = H-1) halved (the stack's s counts it twice).
// GB (FOLD 4, odd modes) = the first-level forward matrix of the DST-I
//    Pm(i, q) = P(i, 2q+1), i, q < h-1 (fold_matrices on size 2H - 1).
// FB (first-level backward, FOLD 2) with its odd-group columns in the level-2
//    position order: FB[r][c] = P(q, fold2_mode(h + c)) for group 1.
// GO (FOLD 4, backward even modes over (sigma, delta)): row r = (b, t): group t/8,
//    output i = 2q + group, q = 8b + t%8 < H; GO[r][c] = P(i, 2c).
// GE (FOLD 2, backward odd modes) = the first-level backward matrix of Pm.
// Layouts as fold_matrices with H for h (GA, GB, GO, GE) and h (FB).
static void fold2_matrices(const std::vector<double>& Pc, int n, int mode, std::vector<double>& ga,
                           std::vector<double>& gb, std::vector<double>& fb, std::vector<double>* go = nullptr,
                           std::vector<double>* ge = nullptr) {
    const int h = (n + 1) / 2, H = h / 2, m = h - 1;
    auto P = [&](int i, int k) { return Pc[(size_t)k * n + i]; };
    {
        const int ld = mode == 0 ? (H + 15) / 16 * 16 : 2 * H;
        ga.assign(mode == 0 ? (size_t)2 * H * ld : (size_t)H * ld, 0.0);
        auto at = [&](int r, int c) -> double& { return mode == 0 ? ga[(size_t)r * ld + c] : ga[(size_t)c * ld + r]; };
        for (int r = 0; r < 2 * H; ++r) {
            const int grp = (r >> 3) & 1, q = (r >> 4) * 8 + (r & 7);
            if (q >= H) continue;
            for (int c = 0; c < H; ++c) {
                const int i = 2 * c + grp;
                at(r, c) = (i == h - 1 ? 0.5 : 1.0) * P(i, 2 * q);
            }
        }
    }
    {
        std::vector<double> Pm((size_t)m * m), unused;
        for (int q = 0; q < m; ++q)
            for (int i = 0; i < m; ++i) Pm[(size_t)q * m + i] = P(i, 2 * q + 1);
        fold_matrices(Pm, m, mode, gb, ge ? *ge : unused);
    }
    if (go) {
        const int ld = mode == 0 ? (H + 15) / 16 * 16 : 2 * H;
        go->assign(mode == 0 ? (size_t)2 * H * ld : (size_t)H * ld, 0.0);
        auto at = [&](int r, int c) -> double& {
            return mode == 0 ? (*go)[(size_t)r * ld + c] : (*go)[(size_t)c * ld + r];
        };
        for (int r = 0; r < 2 * H; ++r) {
            const int grp = (r >> 3) & 1, q = (r >> 4) * 8 + (r & 7);
            if (q >= H) continue;
            for (int c = 0; c < H; ++c) at(r, c) = P(2 * q + grp, 2 * c);
        }
    }
    {
        std::vector<double> ff;
        fold_matrices(Pc, n, mode, ff, fb);
        const int ld = mode == 0 ? (h + 15) / 16 * 16 : 2 * h;
        auto at = [&](int r, int c) -> double& { return mode == 0 ? fb[(size_t)r * ld + c] : fb[(size_t)c * ld + r]; };
        for (int r = 0; r < 2 * h; ++r) {
            const int grp = (r >> 3) & 1, q = (r >> 4) * 8 + (r & 7);
            if (q >= h || grp == 0) continue;
            for (int c = 0; c < h; ++c) {
                const int kb = c < h - 1 ? fold2_mode(h + c, n) : n;
                at(r, c) = (kb < n && q != h - 1) ? P(q, kb) : 0.0;
            }
        }
    }
}

// Fused level-2 backward matrix G6 (etd_back6.cuh) of an axis with n = 4H - 1: 4H
// rows, rounded up to whole 64-row block pairs (H = 8 mod 16: the odd-parity block
// of the last pair), in blocks of 32 (block b: parity par = b & 1, orbit base kb = b >> 1), each
// four 8-row fragments of type t = (r >> 3) & 3 for the orbit k = 16 kb + 2 (r & 7) + par;
// H columns c:
//   t 0  o_k:   P(k, 2c)                        (A: sigma for even k, delta for odd k)
//   t 1  o_c':  P(c', 2c), c' = 2H - 2 - k;  the centre orbit k = H - 1: P(2H - 1, 2c)
//   t 2  eo_k:  P(k, 4c + 1)                    (A: the odd modes 4c + 1 at [2H, 3H))
//   t 3  ee_k:  P(k, 4c + 3), 0 for c = H - 1 and for the centre row k = H - 1
// the same entries GO / GE hold (fold2_matrices), regrouped so one thread gets whole
// orbits.  mode 0 rows contiguous (leading dimension round16(H)); mode 1 [H][4H].
static int back6_rows(int H) { return (4 * H + 63) / 64 * 64; }  // whole (par 0, par 1) block pairs
static void back6_matrix(const std::vector<double>& Pc, int n, int mode, std::vector<double>& g6) {
    const int H = (n + 1) / 4, R = back6_rows(H);
    const int ld = mode == 0 ? (H + 15) / 16 * 16 : R;
    auto P = [&](int i, int k) { return Pc[(size_t)k * n + i]; };
    g6.assign(mode == 0 ? (size_t)R * ld : (size_t)H * ld, 0.0);
    auto at = [&](int r, int c) -> double& { return mode == 0 ? g6[(size_t)r * ld + c] : g6[(size_t)c * ld + r]; };
    for (int r = 0; r < R; ++r) {
        const int blk = r >> 5, t = (r >> 3) & 3, par = blk & 1, kb = blk >> 1;
        const int k = 16 * kb + 2 * (r & 7) + par;
        if (k >= H) continue;
        for (int c = 0; c < H; ++c) {
            double v = 0.0;
            if (t == 0) v = P(k, 2 * c);
            else if (t == 1) v = P(k == H - 1 ? 2 * H - 1 : 2 * H - 2 - k, 2 * c);
            else if (t == 2) v = P(k, 4 * c + 1);
            else if (k != H - 1 && c != H - 1) v = P(k, 4 * c + 3);
            at(r, c) = v;
        }
    }
}

// Device bytes build_plan allocates (the memory guard and etd_plan_device_bytes):
// state x2 (ns fields on the level-2 schedule, else 2 ns) + Z + W at 2 ns fields each; sharded: send blocks (ns fields), the
// z-stage blocks zin/Zz/Wz (2 ns fields of this rank's y rows, full z) and the
// receive blocks (2 ns fields); per axis P and P^T plus the split matrices
// (<= 6 npad^2); Thomas factors and checkpoints; 64 MiB for descriptors,
// d-vectors, tables and the allocator's rounding.
// Whether a plan runs the second-level split schedule on every axis (the decision
// build_plan makes, restated from the desc and the A/B environment switches): its
// source pass writes the first transform's stack into scratch, so the state
// buffers need no f slots (ns fields instead of [U,(V),fU,(fV)]).
static bool level2_schedule(const etd_desc& d) {
    if (d.backend == ETD_THOMAS) return false;
    auto env_is = [](const char* k, char c) { const char* e = std::getenv(k); return e && e[0] == c; };
    if (env_is("ETD_DENSE", '1') || env_is("ETD_FUSED_SOURCE", '1') || env_is("ETD_FOLD2", '0')) return false;
    const char* fa = std::getenv("ETD_FOLD_AXES");
    const int axes = fa ? std::atoi(fa) : 7;
    const double npts = (double)d.n[0] * d.n[1] * (d.dim == 3 ? d.n[2] : 1);
    if (!(env_is("ETD_FOLD2", '1') || npts >= 262144.0)) return false;
    for (int a = 0; a < d.dim; ++a) {
        const int h = (d.n[a] + 1) / 2;
        if (!(h % 16 == 0 && (d.n[a] & 1) && (axes >> a & 1))) return false;
    }
    return true;
}

static unsigned long long plan_device_bytes(const etd_desc& d) {
    const int G = d.world_size < 1 ? 1 : d.world_size;
    const int nz = d.dim == 3 ? d.n[2] : 1;
    const unsigned long long pitch = (unsigned long long)round_up(d.n[0], 32);
    int z0 = 0, z1 = nz, j0 = 0, j1 = d.n[1];
    if (G > 1) {
        partition(nz, G, d.rank, z0, z1);
        partition(d.n[1], G, d.rank, j0, j1);
    }
    const unsigned long long F = pitch * d.n[1] * (z1 - z0), ns = d.nspecies;
    const unsigned long long sf = level2_schedule(d) ? ns : 2 * ns;  // fields per state buffer
    unsigned long long b = (2ull * sf + 2ull * 2 * ns) * F * 8;
    if (G > 1) {
        const unsigned long long Fz = pitch * (j1 - j0) * nz;
        b += F * ns * 8 + 3ull * Fz * 2 * ns * 8 + F * 2 * ns * 8;
    }
    for (int a = 0; a < d.dim; ++a) {
        const unsigned long long np = (unsigned long long)round_up(d.n[a], 32);
        b += d.backend == ETD_THOMAS ? 2ull * 3 * ns * d.n[a] * 16 : 6ull * np * np * 8;
    }
    if (d.backend == ETD_THOMAS) b += F * ns * 2 * 16 / 4;  // checkpoint scratch (2/K complex per point)
    return b + (64ull << 20);
}

static void memory_guard(const etd_desc& d) {
    const unsigned long long need = plan_device_bytes(d);
    if (d.memory_cap_bytes && need > d.memory_cap_bytes)
        throw MemoryGuardError("device plan needs " + std::to_string(need >> 20) + " MiB, above the " +
                               std::to_string(d.memory_cap_bytes >> 20) + " MiB cap");
    size_t freeb = 0, total = 0;
    ETD_CK(cudaMemGetInfo(&freeb, &total));
    if (need > freeb)
        throw MemoryGuardError("device plan needs " + std::to_string(need >> 20) + " MiB on rank " +
                               std::to_string(d.world_size > 1 ? d.rank : 0) + ", " + std::to_string(freeb >> 20) +
                               " MiB free on device " + std::to_string(d.device) +
                               (d.dim == 3 ? " (shard the z-slabs over more GPUs: world_size)" : ""));
}

static void build_plan(Plan& p, const etd_desc& d) {
    validate(d);
    p.d = d;
    const bool sys = d.nspecies == 2;
    p.dim = d.dim;
    p.ns = d.nspecies;
    p.tau = d.tau;
    p.G = d.world_size < 1 ? 1 : d.world_size;
    p.rank = p.G > 1 ? d.rank : 0;
    p.sharded = p.G > 1;
    p.local_group = p.sharded && d.nccl_unique_id == nullptr;
    int dev_count = 0;
    if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0)
        throw NoDevice("no CUDA device visible: the ETD2RK-DS CUDA backend has no CPU fallback");
    ETD_CK(cudaSetDevice(d.device));
    int major = 0;
    ETD_CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d.device));
    if (major != 10) throw NoDevice("this build targets sm_100a (B200)");
    ETD_CK(cudaDeviceGetAttribute(&p.nsm, cudaDevAttrMultiProcessorCount, d.device));
    memory_guard(d);

    p.nx = d.n[0];
    p.ny = d.n[1];
    p.nz = d.dim == 3 ? d.n[2] : 1;
    p.pitch = round_up(p.nx, 32);
    p.dmax = 0;
    for (int a = 0; a < d.dim; ++a) {
        p.npad[a] = round_up(d.n[a], 32);
        p.dmax = std::max(p.dmax, p.npad[a]);
    }
    p.zlo.resize(p.G); p.zhi.resize(p.G); p.jlo.resize(p.G); p.jhi.resize(p.G);
    for (int r = 0; r < p.G; ++r) {
        partition(p.nz, p.G, r, p.zlo[r], p.zhi[r]);
        partition(p.ny, p.G, r, p.jlo[r], p.jhi[r]);
    }
    const int R = p.rank;
    p.slab = View{p.nx, p.ny, p.zhi[R] - p.zlo[R], p.pitch, p.pitch * p.ny, 0, 0, p.zlo[R]};
    p.slab.F = p.slab.plane * p.slab.nz;
    if (p.sharded) {
        p.zC = kZChunks;
        if (const char* e = std::getenv("ETD_ZCHUNKS")) p.zC = std::max(1, std::atoi(e));
        const ZChunks zc = zchunks(p.ny, p.nz, p.ns, p.G, p.pitch, p.zC);
        for (int k = 0; k < p.zC; ++k) {
            int a, b;
            zc.rows(R, k, a, b);
            View v{p.nx, b - a, p.nz, p.pitch, p.pitch * (b - a), 0, p.jlo[R] + a, 0};
            v.F = v.plane * v.nz;
            p.zch.push_back(v);
            p.zbase.push_back(zc.base(R, k));
        }
    }

    ETD_CK(cudaStreamCreateWithFlags(&p.stream, cudaStreamNonBlocking));
    auto alloc = [&](double*& ptr, size_t elems) {
        ETD_CK(cudaMalloc(&ptr, elems * sizeof(double)));
        ETD_CK(cudaMemsetAsync(ptr, 0, elems * sizeof(double), p.stream));  // pads stay +0.0 forever
    };
    const size_t F = (size_t)p.slab.F;
    // [U,(V),fU,(fV)]; the level-2 schedule's source pass writes f into the first
    // transform's stack in scratch, so its state buffers hold only U(,V)
    p.state_fields = level2_schedule(d) ? p.ns : 2 * p.ns;
    for (int s = 0; s < 2; ++s) alloc(p.state[s], F * p.state_fields);
    alloc(p.Z, F * 2 * p.ns);
    alloc(p.W, F * 2 * p.ns);
    if (p.sharded) {
        const size_t Fz = (size_t)p.pitch * (p.jhi[R] - p.jlo[R]) * p.nz;
        alloc(p.sendbuf, F * p.ns);
        alloc(p.zin, Fz * 2 * p.ns);
        alloc(p.Zz, Fz * 2 * p.ns);
        alloc(p.Wz, Fz * 2 * p.ns);
        alloc(p.recvb, F * 2 * p.ns);
        ETD_CK(cudaMalloc(&p.codes, sizeof(int) * (p.G + 1)));
        ETD_CK(cudaMemsetAsync(p.codes, 0, sizeof(int) * (p.G + 1), p.stream));
    }

    // per-axis eigensystems and d-vectors (stepper.cpp:118-177; systems use the
    // unit-kappa operator and kappa_c * lambda, system_stepper.cpp:47-61)
    const bool exact = d.family == ETD_EXACT;
    const PadeScheme scheme = pade_scheme(exact ? 0 : d.family);
    p.thomas = d.backend == ETD_THOMAS;
    std::vector<double> hd((size_t)3 * 3 * 9 * 2 * p.dmax, 0.0);
    // Parity split on every spectral axis whose half extent h = (n+1)/2 is a
    // multiple of 8 (n = 16m - 1 or 16m: all BASELINE configs); ETD_DENSE=1 turns
    // it off.  A fused source prologue (ETD_FUSED_SOURCE=1) keeps its axis dense.
    {
        const char* dn = std::getenv("ETD_DENSE");
        const bool dense_env = dn && dn[0] == '1';
        const char* fenv0 = std::getenv("ETD_FUSED_SOURCE");
        const bool fused0 = fenv0 && fenv0[0] == '1';
        const char* fa = std::getenv("ETD_FOLD_AXES");  // bit mask (tests / dev tools)
        const int axes = fa ? std::atoi(fa) : 7;
        for (int a = 0; a < d.dim; ++a) {
            const int h = (d.n[a] + 1) / 2;
            p.fh[a] = h;
            p.fold[a] = !p.thomas && !dense_env && h % 8 == 0 && (axes >> a & 1) &&
                        !(fused0 && a == (d.dim == 3 ? 2 : 1));
        }
        // Second-level split where n = 4H - 1 with H a multiple of 8
        // (n = 32m - 1: every BASELINE config); the step uses it when every axis has
        // it and the grid has >= 2^18 points (below, its extra stack-pass launches
        // cost more than the halved contractions save: config 0, 127^2, runs
        // 0.066 ms/step first-level vs 0.152 ms second-level; config 1, 1023^2,
        // 0.405 vs 0.358).  ETD_FOLD2=0 turns it off, =1 forces it on any size.
        const char* f2 = std::getenv("ETD_FOLD2");
        const bool f2_off = f2 && f2[0] == '0', f2_force = f2 && f2[0] == '1';
        const double npts = (double)d.n[0] * d.n[1] * (d.dim == 3 ? d.n[2] : 1);
        p.fold2_all = !f2_off && !fused0 && (f2_force || npts >= 262144.0);
        for (int a = 0; a < d.dim; ++a) {
            p.fold2[a] = p.fold[a] && !f2_off && (d.n[a] & 1) && p.fh[a] % 16 == 0;
            p.fold2_all = p.fold2_all && p.fold2[a];
        }
        // mixed levels are not scheduled: every axis keeps §4a then
        for (int a = 0; a < d.dim; ++a) p.fold2[a] = p.fold2[a] && p.fold2_all;
        if (p.fold2_all != level2_schedule(d))
            throw ConfigError("internal: level-2 schedule decision differs from the state allocation");
        // level-2 backward transforms fused into one launch each;
        // ETD_BACK6=0 keeps the two launches + etd_unfold2 pass of round 1 (A/B, tests)
        const char* b6 = std::getenv("ETD_BACK6");
        p.back6 = p.fold2_all && !(b6 && b6[0] == '0');
    }
    for (int a = 0; a < d.dim && p.thomas; ++a) {
        // build_thomas_payload (thomas.cpp:88-126) per species: c = tau diag k - s_l,
        // e = tau off k; systems scale the unit-kappa operator by kappa_c
        // (system_stepper.cpp:62-64)
        const int n = d.n[a];
        const AxisOperator op = axis_operator(n, d.low[a], d.high[a], d.dim, sys ? 1.0 : d.kappa[0], d.q);
        const auto& poles = scheme.terms[0];
        const int np = (int)poles.size();
        if (np > 2) throw ConfigError("Thomas backend: at most 2 poles");
        std::vector<double2> hf((size_t)p.ns * np * 3 * n);
        ThomasArgs& tb = p.thbase[a];
        tb = ThomasArgs{};
        tb.F = p.slab.F;
        tb.n = n;
        tb.ns = p.ns;
        tb.npoles = np;
        tb.tau = d.tau;
        tb.ny = p.slab.ny;
        tb.gj0 = p.slab.gj0;
        tb.gz0 = p.slab.gz0;
        for (int i = 0; i < 8; ++i) tb.sp[i] = d.src_params[i];
        for (int c = 0; c < p.ns; ++c) {
            const double ks = sys ? d.kappa[c] : 1.0;
            const std::complex<double> e(d.tau * op.off * ks, 0.0);
            tb.e[c] = make_double2(e.real(), e.imag());
            for (int l = 0; l < np; ++l) {
                const std::complex<double> cc = d.tau * op.diag * ks - poles[l].pole;
                const ThomasPole f = thomas_factor(n, cc, e);
                double2* o = hf.data() + ((size_t)c * np + l) * 3 * n;
                for (int i = 0; i < n; ++i) {
                    o[i] = make_double2(f.mul[i].real(), f.mul[i].imag());
                    o[n + i] = make_double2(f.piv[i].real(), f.piv[i].imag());
                    o[2 * n + i] = make_double2(f.inv[i].real(), f.inv[i].imag());
                }
                for (int ell = 1; ell <= 3; ++ell) {
                    const auto& t = scheme.terms[ell - 1];
                    if ((int)t.size() != np || t[l].pole != poles[l].pole)
                        throw NumericsError("pole ordering differs across weight functions");
                    tb.res[c][ell - 1][l] = make_double2(t[l].residue.real(), t[l].residue.imag());
                }
            }
        }
        // padded by one stage of rows: the kernels stage factor slices [jt J, jt J + J)
        ETD_CK(cudaMalloc(&p.thfac[a], (hf.size() + 64) * sizeof(double2)));
        ETD_CK(cudaMemset(p.thfac[a], 0, (hf.size() + 64) * sizeof(double2)));
        ETD_CK(cudaMemcpy(p.thfac[a], hf.data(), hf.size() * sizeof(double2), cudaMemcpyHostToDevice));
        tb.fac = p.thfac[a];
    }
    for (int a = 0; a < d.dim && !p.thomas; ++a) {
        const int n = d.n[a], np = p.npad[a];
        const AxisOperator op = axis_operator(n, d.low[a], d.high[a], d.dim, sys ? 1.0 : d.kappa[0], d.q);
        std::vector<double> Pc, lam, fb2_tmp;
        eigensystem(op, Pc, lam);
        std::vector<double> pr((size_t)np * np, 0.0), ptr((size_t)np * np, 0.0);
        for (int i = 0; i < n; ++i)
            for (int kk = 0; kk < n; ++kk) {
                pr[(size_t)i * np + kk] = Pc[(size_t)kk * n + i];   // P(i,kk) row-major
                ptr[(size_t)i * np + kk] = Pc[(size_t)i * n + kk];  // P(kk,i) = P^T row-major
            }
        ETD_CK(cudaMalloc(&p.PR[a], pr.size() * 8));
        ETD_CK(cudaMalloc(&p.PTR[a], ptr.size() * 8));
        ETD_CK(cudaMemcpy(p.PR[a], pr.data(), pr.size() * 8, cudaMemcpyHostToDevice));
        ETD_CK(cudaMemcpy(p.PTR[a], ptr.data(), ptr.size() * 8, cudaMemcpyHostToDevice));
        if (p.fold2[a] && p.back6) {
            std::vector<double> g6;
            back6_matrix(Pc, n, a == 0 ? 0 : 1, g6);
            ETD_CK(cudaMalloc(&p.G6[a], g6.size() * 8));
            ETD_CK(cudaMemcpy(p.G6[a], g6.data(), g6.size() * 8, cudaMemcpyHostToDevice));
        }
        if (p.fold2[a]) {
            std::vector<double> ga, gb, go, ge;
            fold2_matrices(Pc, n, a == 0 ? 0 : 1, ga, gb, fb2_tmp, &go, &ge);
            for (auto [dst, v] : {std::pair{&p.GA[a], &ga}, std::pair{&p.GB[a], &gb}, std::pair{&p.GO[a], &go},
                                  std::pair{&p.GE[a], &ge}}) {
                ETD_CK(cudaMalloc(dst, v->size() * 8));
                ETD_CK(cudaMemcpy(*dst, v->data(), v->size() * 8, cudaMemcpyHostToDevice));
            }
        }
        if (p.fold[a]) {
            std::vector<double> ff, fb;
            fold_matrices(Pc, n, a == 0 ? 0 : 1, ff, fb);
            if (p.fold2[a]) fb.swap(fb2_tmp);  // backward reads the level-2 mode positions
            ETD_CK(cudaMalloc(&p.FF[a], ff.size() * 8));
            ETD_CK(cudaMalloc(&p.FB[a], fb.size() * 8));
            ETD_CK(cudaMemcpy(p.FF[a], ff.data(), ff.size() * 8, cudaMemcpyHostToDevice));
            ETD_CK(cudaMemcpy(p.FB[a], fb.data(), fb.size() * 8, cudaMemcpyHostToDevice));
        }
        for (int c = 0; c < p.ns; ++c) {
            std::vector<double> lc(lam);
            if (sys)
                for (auto& x : lc) x *= d.kappa[c];
            // natural order, and parity-major (position q < h: mode 2q; h + q: mode 2q + 1)
            const int h = p.fh[a];
            auto put = [&](int slot, const std::vector<double>& v, double sc) {
                double* o = hd.data() + (((size_t)a * 9 + slot) * 2 + c) * p.dmax;
                double* op = hd.data() + (((size_t)(3 + a) * 9 + slot) * 2 + c) * p.dmax;
                double* o2 = hd.data() + (((size_t)(6 + a) * 9 + slot) * 2 + c) * p.dmax;
                for (int i = 0; i < n; ++i) o[i] = sc * v[i];
                for (int pos = 0; pos < n; ++pos) {
                    const int k = pos < h ? 2 * pos : 2 * (pos - h) + 1;
                    op[pos] = k < n ? sc * v[k] : 0.0;
                    if (p.fold2[a]) {
                        const int k2 = fold2_mode(pos, n);
                        o2[pos] = k2 < n ? sc * v[k2] : 0.0;
                    }
                }
            };
            if (exact) {
                // BackendKind::ExactExpReference (stepper.cpp:145-170, 259-295): the same
                // step structure with exact exponential multipliers e^{-tau lambda}
                // (every axis), tau phi1(tau lambda) and tau phi2(tau lambda) (x axis).
                // The reference caps this dense path at 64 points per axis; the
                // transform engine has no such limit.
                const auto ev = exp_multipliers(lc, d.tau);
                const auto g1 = phi_multipliers(lc, d.tau, 1), hh = phi_multipliers(lc, d.tau, 2);
                put(0, ev, 1.0); put(1, g1, 1.0); put(2, hh, 1.0);
                put(3, ev, 1.0); put(4, g1, 1.0); put(5, hh, 1.0);
                put(6, ev, 2.0); put(7, g1, 2.0); put(8, hh, 2.0);
                continue;
            }
            const auto d1 = dvector(lc, d.tau, scheme, 1), d2 = dvector(lc, d.tau, scheme, 2),
                       d3 = dvector(lc, d.tau, scheme, 3);
            // production slots (power-of-two 2 folds exactly; tau folds once)
            put(0, d1, 2.0);
            put(1, d2, 2.0 * d.tau);
            put(2, d3, 2.0 * d.tau);
            // raw and 2x slots for kernel-level tests
            put(3, d1, 1.0); put(4, d2, 1.0); put(5, d3, 1.0);
            put(6, d1, 2.0); put(7, d2, 2.0); put(8, d3, 2.0);
        }
    }
    // sin(pi x_i) tables, reference expression std::sin(pi * coord(a, i)) with
    // coord = low + (i+1) h (grid.hpp:36, problems.cpp:22-23)
    for (int a = 0; a < d.dim; ++a) {
        const double h = (d.high[a] - d.low[a]) / (d.n[a] + 1);
        std::vector<double> st(d.n[a]);
        for (int i = 0; i < d.n[a]; ++i) st[i] = std::sin(std::numbers::pi * (d.low[a] + (i + 1) * h));
        ETD_CK(cudaMalloc(&p.sintab[a], st.size() * 8));
        ETD_CK(cudaMemcpy(p.sintab[a], st.data(), st.size() * 8, cudaMemcpyHostToDevice));
    }
    ETD_CK(cudaMalloc(&p.dvec, hd.size() * 8));
    ETD_CK(cudaMemcpy(p.dvec, hd.data(), hd.size() * 8, cudaMemcpyHostToDevice));
    ETD_CK(cudaMalloc(&p.status, sizeof(StepStatus)));
    ETD_CK(cudaMallocHost(&p.status_host, sizeof(StepStatus)));
    std::memset(p.status_host, 0, sizeof(StepStatus));
    ETD_CK(cudaMemcpy(p.status, p.status_host, sizeof(StepStatus), cudaMemcpyHostToDevice));
    if (p.thomas) {
        for (int a = 0; a < d.dim; ++a) {
            p.thbase[a].sinx = p.sintab[0];
            p.thbase[a].siny = p.sintab[1];
            p.thbase[a].sinz = d.dim == 3 ? p.sintab[2] : nullptr;
            p.thbase[a].status = p.status;
        }

    }

    // opt every variant into large dynamic shared memory
    static bool attr_done = false;
    if (!attr_done) {
        for (int mode = 0; mode < 2; ++mode)
            for (int S : {1, 2, 4})
                for (int e = 0; e < 6; ++e)
                    for (int pro = 0; pro < 2; ++pro)
                        for (int sk : {0, 1, 2, 3, 4, 5, 10, 11, 12, 13})
                            for (int tile = 0; tile < 4; ++tile)
                                for (int fold = 0; fold < 7; ++fold) {
                                    try {
                                        KernelSpec ks = pick(mode, S, e, pro != 0, sk, tile, fold);
                                        ETD_CK(cudaFuncSetAttribute(
                                            ks.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            std::getenv("ETD_ONE_CTA") ? std::max(ks.smem, 120000) : ks.smem));
                                    } catch (const ConfigError&) {
                                    }
                                }
        attr_done = true;
    }

    if (p.sharded && !p.local_group) {
        auto& nc = Nccl::get();
        ncclUniqueId id;
        std::memcpy(&id, d.nccl_unique_id, sizeof(id));
        nc.check(nc.CommInitRank(&p.comm, p.G, id, p.rank), "ncclCommInitRank");
    }

    // ---- step schedule per state parity ----
    const int ns = p.ns;
    const char* fenv = std::getenv("ETD_FUSED_SOURCE");
    const bool fused = fenv && fenv[0] == '1';
    const View& V = p.slab;
    for (int par = 0; par < 2; ++par) {
        auto& L = p.steps[par];
        L.clear();
        const double* in = p.state[par];
        double* out = p.state[1 - par];
        if (p.thomas) {
            // BackendKind::Thomas (stepper.cpp:231-240, 243-253; system_stepper.cpp:74-114):
            // fn = f(t, U); w = Q1_y(Q1_z(.)) of [U, fn]; What = Q1_x(w1) + tau Q2_x(w2);
            // fw = f(t + tau, What) - w2; U1 = What + tau Q3_x(fw)
            const long long F = V.F;
            (void)F;
            L.push_back(p.source_op(V, const_cast<double*>(in)));
            const double* yin = in;
            if (p.dim == 3) {
                L.push_back(p.thomas_op("thomas_z", 2, TH_STORE, in, p.Z, 2 * ns, 1));
                yin = p.Z;
            }
            L.push_back(p.thomas_op("thomas_y", 1, TH_STORE, yin, p.W, 2 * ns, 1));
            L.push_back(p.thomas_op("thomas_x_what", 0, TH_WHAT, p.W, p.Z, 2 * ns, 1));
            L.push_back(p.thomas_op("thomas_x_upd", 0, TH_UPDATE, p.Z, out, ns, 3, 0, ns));
            continue;
        }
        // The source f(t, U) either runs as its own HBM-bound pass into the f
        // slots of the state stack (default; "source" + "z_fwd"/"y_fwd"), or fused
        // into the first transform's prologue (ETD_FUSED_SOURCE=1, "z_fwd_src"):
        // measured 265 vs 246 + 5.5 ms per config-4 step.
        // A parity-split first axis gets its stack folded by the source pass (into
        // `scratch`, free until the axis' backward transform writes it), so the
        // forward transform runs FOLD 4 with no s/d adds in its main loop.
        // Second-level split (p.fold2_all): every forward transform is
        // an etd_fold2 stack (src -> tmp) and its even/odd-mode launches (tmp -> dst).
        const bool f2 = p.fold2_all;
        bool zy_fused = false;  // unsharded 3D level 2: z_back's unfold + the y stack in one pass
        // S = 4 transform launches as two S = 2 launches (2 CTAs/SM overlap one CTA's
        // epilogue with the other's main loop; config 4 529.8 -> 521.1 ms/step,
        // config 3 42.0 -> 40.0); ETD_PAIRS=0 keeps the S = 4 launches
        const char* pe = std::getenv("ETD_PAIRS");
        const bool pairs = !(pe && pe[0] == '0');
        auto fwd2 = [&](const View& vv, const std::string& nm, int axis, int S, int epi, const double* src,
                        double* tmp, double* dst, bool from1, const double* dA, const double* dB = nullptr,
                        const double* aux = nullptr, bool stacked = false) {
            if (!stacked) L.push_back(p.fold_op(vv, "fold_" + nm, axis, src, tmp, S, from1));
            const long long F = vv.F;
            for (int part = 1; part <= 2; ++part) {
                const std::string pn = nm + (part == 1 ? "_even" : "_odd");
                if (pairs && S == 4) {
                    // two S = 2 launches (2 CTAs/SM): fields (0,1), (2,3); the mix pairs
                    // each species' (w1, w2) = fields (c, c + 2)
                    for (int h2 = 0; h2 < 2; ++h2) {
                        const bool mix = epi == EPI_MIX;
                        const long long off = mix ? h2 * F : 2 * h2 * F;
                        L.push_back(kernel_op(p.transform(vv, pn + (h2 ? "_b" : "_a"), axis, false, 2, epi, false,
                                                          tmp + off, dst + off, false, nullptr, false, part,
                                                          mix ? 2 * F : 0)));
                        L.back().L.args.dA = dA + (mix ? h2 * p.dmax : 0);
                        L.back().L.args.dB = dB ? dB + (mix ? h2 * p.dmax : 0) : nullptr;
                        L.back().L.args.aux = aux;
                    }
                    continue;
                }
                L.push_back(kernel_op(p.transform(vv, pn, axis, false, S, epi, false, tmp, dst, false, nullptr,
                                                  false, part)));
                L.back().L.args.dA = dA;
                L.back().L.args.dB = dB;
                L.back().L.args.aux = aux;
            }
        };
        // ... and every backward transform two launches into an intermediate stack
        // (in -> tmp) finished by etd_unfold2 (tmp -> out) with the stage epilogue.
        // With p.back6 it is ONE fused launch (etd_back6: all four quarters, butterflies
        // and the stage epilogue on the accumulators) straight from src to dst (src !=
        // dst; tmp unused); S = 4 stacks run as two S = 2 launches.
        auto back2 = [&](const View& vv, const std::string& nm, int axis, int S, const double* src, double* tmp,
                         double* dst, int uf, const double* aux = nullptr, double* fout = nullptr) {
            if (p.back6) {
                if (src == dst) throw ConfigError("internal: fused backward in place");
                const int epi = uf == UF_UPDATE ? EPI_UPDATE : uf == UF_WHAT_SRC ? EPI_WHAT_SRC : EPI_STORE;
                // y/z: one launch per field (S = 1 tiles are 64 x wide, so a warp holds 16 x and
                // the XPAIR fragment interleave gives 16-byte LDS / stores); ETD_BACK6_XPAIR=0:
                // S = 4 stacks as two S = 2 launches (A/B)
                const int nl = (back6_xpair() && axis != 0) ? S : (S == 4 ? 2 : 1);
                const int per = S / nl;
                for (int h2 = 0; h2 < nl; ++h2) {
                    const std::string sfx(1, (char)('a' + h2));
                    L.push_back(kernel_op(p.transform(vv, nl >= 2 ? nm + "_" + sfx : nm, axis, true, per,
                                                      epi, false, src + (size_t)per * h2 * vv.F,
                                                      dst + (size_t)per * h2 * vv.F, false,
                                                      nullptr, false, 6)));
                    L.back().L.args.aux = aux;
                    L.back().L.args.fout = fout;
                }
                return;
            }
            for (int part = 3; part <= 4; ++part) {
                const std::string pn = nm + (part == 3 ? "_o" : "_e");
                if (pairs && S == 4) {
                    for (int h2 = 0; h2 < 2; ++h2)
                        L.push_back(kernel_op(p.transform(vv, pn + (h2 ? "_b" : "_a"), axis, true, 2, EPI_STORE,
                                                          false, src + 2 * h2 * vv.F, tmp + 2 * h2 * vv.F, false,
                                                          nullptr, false, part)));
                    continue;
                }
                L.push_back(kernel_op(p.transform(vv, pn, axis, true, S, EPI_STORE, false, src, tmp, false, nullptr,
                                                  false, part)));
            }
            L.push_back(p.unfold_op(vv, nm, axis, uf, tmp, dst, S, aux, fout));
        };
        auto first_transform = [&](const View& vv, int axis, double* stack, double* dst, double* scratch) {
            if (f2) {
                // the source pass writes [U,(V),fU,(fV)]'s level-2 stack along the axis
                L.push_back(p.source_op(vv, stack, scratch, axis, true));
                fwd2(vv, axis == 2 ? "z_fwd" : "y_fwd", axis, 2 * ns, EPI_SCALE, stack, scratch, dst, false,
                     p.dv(axis, 0), nullptr, nullptr, true);
                return;
            }
            const char* nm = axis == 2 ? (fused ? "z_fwd_src" : "z_fwd") : (fused ? "y_fwd_src" : "y_fwd");
            const bool pf = !fused && p.fold[axis];
            if (!fused) L.push_back(p.source_op(vv, stack, pf ? scratch : nullptr, pf ? axis : 0));
            L.push_back(kernel_op(p.transform(vv, nm, axis, false, 2 * ns, EPI_SCALE, fused, pf ? scratch : stack,
                                              dst, false, nullptr, pf)));
            L.back().L.args.dA = p.dv(axis, 0);
        };
        if (p.dim == 3 && !p.sharded) {
            first_transform(V, 2, const_cast<double*>(in), p.Z, p.W);
            if (f2 && p.back6) {
                // z_back fused (Z -> W physical), then the y stack pass (W -> Z)
                back2(V, "z_back", 2, 2 * ns, p.Z, nullptr, p.W, UF_STORE);
                L.push_back(p.fold_op(V, "fold_y_fwd", 1, p.W, p.Z, 2 * ns));
                zy_fused = true;
            } else if (f2) {
                // z_back's launches (Z -> W), then its unfold fused with the y stack (W -> Z)
                const bool pr = pairs && 2 * ns == 4;
                for (int part = 3; part <= 4; ++part) {
                    const std::string pn = std::string("z_back") + (part == 3 ? "_o" : "_e");
                    for (int h2 = 0; h2 < (pr ? 2 : 1); ++h2)
                        L.push_back(kernel_op(p.transform(V, pr ? pn + (h2 ? "_b" : "_a") : pn, 2, true,
                                                          pr ? 2 : 2 * ns, EPI_STORE, false,
                                                          p.Z + 2 * h2 * V.F, p.W + 2 * h2 * V.F, false, nullptr,
                                                          false, part)));
                }
                Op zy;
                zy.kind = Op::ZYFOLD;
                zy.name = zy.L.name = "z_back_y_stack";
                zy.L.mode = 1;
                zy.zargs = ZYArgs{p.W, p.Z, (long long)V.F, V.pitch, V.plane, 2 * ns, V.nx, V.ny, V.nz,
                                  p.fh[2] / 2, p.fh[1] / 2, 0, V.nx};
                // etd_unfold_fold_zy moves two fields per work item (f0, f0 + 1)
                if (zy.zargs.nf % 2 != 0) throw ConfigError("internal: z_back_y_stack needs an even field count");
                zy.src_blocks = 148u * 16u;
                zy.L.bytes = (double)V.nx * V.ny * V.nz * 8.0 * 2 * 2 * ns;
                L.push_back(zy);
                zy_fused = true;
            } else {
                L.push_back(kernel_op(p.transform(V, "z_back", 2, true, 2 * ns, EPI_STORE, false, p.Z, p.W)));
            }
        } else if (p.dim == 3) {
            // ---- z stage on y-row chunks: pack; forward exchanges (comm stream);
            // per chunk source + z transforms (compute stream) overlapping the next
            // chunk's forward and the previous chunk's backward exchange; unpack ----
            const int C = p.zC;
            const int EV_PACK = 0, EV_B = 1;
            auto EV_F = [&](int k) { return 2 + k; };
            auto EV_Z = [&](int k) { return 2 + C + k; };
            const auto sched = sharded_schedule(p.nx, p.ny, p.nz, ns, p.G, p.rank, p.pitch, C);
            double* bufs[6] = {const_cast<double*>(in), p.sendbuf, p.zin, p.Wz, p.recvb, p.W};
            auto exchange = [&](int phase, int k, const char* name) {
                Op ex;
                ex.kind = Op::EXCHANGE;
                ex.name = name;
                ex.strm = 1;
                for (const auto& r : sched) {
                    if (r.phase != phase || r.chunk != k) continue;
                    if (r.kind == SK_SEND)
                        ex.sends.push_back({(int)r.peer, bufs[r.sbuf] + r.soff, (size_t)r.count * 8});
                    else if (r.kind == SK_RECV)
                        ex.recvs.push_back({(int)r.peer, bufs[r.dbuf] + r.doff, (size_t)r.count * 8});
                }
                return ex;
            };
            auto copies = [&](int phase, const char* name) {
                const size_t first = L.size();
                for (const auto& r : sched)
                    if (r.phase == phase && r.kind == SK_COPY)
                        L.push_back(copy_op(name, bufs[r.dbuf] + r.doff, r.dpitch * 8, bufs[r.sbuf] + r.soff,
                                            r.spitch * 8, r.width * 8, r.height));
                return first;
            };
            copies(SP_PACK, "pack");
            L.back().rec_ev = EV_PACK;
            for (int k = 0; k < C; ++k) {
                Op f = exchange(SP_FWD, k, "a2a_fwd");
                if (k == 0) f.wait_ev = EV_PACK;
                f.rec_ev = EV_F(k);
                L.push_back(f);
            }
            // ops a populated chunk emits: source (unless fused) + z_fwd launches + z_back
            // launches (+ the level-2 unfold); an empty chunk pads with as many no-ops so
            // every rank's op list stays aligned with rank 0's (group_steps, NCCL groups)
            const int zl = (f2 && (pairs || p.back6) && 2 * ns == 4) ? 2 : 1;  // launches per level-2 part
            const int zb6 = back6_xpair() ? 2 * ns : zl;  // fused backward launches of a chunk
            const int chunk_ops = fused ? 2 : f2 ? 1 + 2 * zl + (p.back6 ? zb6 : 2 * zl + 1) : 3;
            for (int k = 0; k < C; ++k) {
                const View& vk = p.zch[k];
                const size_t first = L.size();
                if (vk.ny > 0) {
                    double* zin_k = p.zin + p.zbase[k];
                    double* zz_k = p.Zz + p.zbase[k];
                    double* wz_k = p.Wz + p.zbase[k];
                    first_transform(vk, 2, zin_k, zz_k, wz_k);
                    if (f2) back2(vk, "z_back", 2, 2 * ns, zz_k, zin_k, wz_k, UF_STORE);
                    else L.push_back(kernel_op(p.transform(vk, "z_back", 2, true, 2 * ns, EPI_STORE, false, zz_k, wz_k)));
                    if ((int)(L.size() - first) != chunk_ops)
                        throw ConfigError("internal: z-chunk op count " + std::to_string(L.size() - first) +
                                          " != " + std::to_string(chunk_ops));
                } else {
                    // an empty chunk keeps the op list aligned across virtual ranks
                    for (int i = 0; i < chunk_ops; ++i) {
                        Op o;
                        o.kind = Op::NOP;
                        o.name = "z_empty";
                        L.push_back(o);
                    }
                }
                L[first].wait_ev = EV_F(k);
                L.back().rec_ev = EV_Z(k);
                Op b = exchange(SP_BACK, k, "a2a_back");
                b.wait_ev = EV_Z(k);
                b.rec_ev = EV_B;
                L.push_back(b);
            }
            if (f2 && p.back6) {
                // the unpack fused into the y stack pass: it reads the slab's y rows
                // straight from the receive blocks (recv_row_table) and writes the y
                // stack into Z, as the unsharded z_back + fold_y_fwd do
                if (!p.recv_rows) {  // (both step parities share it)
                    const auto tab = recv_row_table(p.ny, p.nz, ns, p.G, p.rank, p.pitch, C);
                    ETD_CK(cudaMalloc(&p.recv_rows, tab.size() * sizeof(long long)));
                    ETD_CK(cudaMemcpy(p.recv_rows, tab.data(), tab.size() * sizeof(long long),
                                      cudaMemcpyHostToDevice));
                }
                Op fy = p.fold_op(V, "fold_y_fwd", 1, p.recvb, p.Z, 2 * ns);
                fy.fargs.rows = p.recv_rows;
                fy.wait_ev = EV_B;
                L.push_back(fy);
                zy_fused = true;
            } else {
                L[copies(SP_UNPACK, "unpack")].wait_ev = EV_B;
            }
        }
        if (f2) {
            // y stage on (B1, B2) with the z-filtered stack (3D) in B2, then the x stage
            // on (Xa, Xb) = (B2, B1); the z stage left its output in Z (unsharded) or the
            // unpack in W (sharded)
            double *B1 = p.W, *B2 = p.Z;
            if (zy_fused) {
                // the y stack is already in Z: y_fwd Z -> W, y_back W -> (Z) -> W
                B1 = p.Z, B2 = p.W;
                fwd2(V, "y_fwd", 1, 2 * ns, EPI_SCALE, nullptr, B1, B2, false, p.dv(1, 0), nullptr, nullptr, true);
            } else if (p.dim == 3) {
                if (p.sharded) B1 = p.Z, B2 = p.W;
                fwd2(V, "y_fwd", 1, 2 * ns, EPI_SCALE, B2, B1, B2, false, p.dv(1, 0));
            } else {
                first_transform(V, 1, const_cast<double*>(in), B2, B1);
            }
            const size_t Fs = (size_t)ns * V.F;
            if (p.back6) {
                // fused backward launches never run in place:
                //   y_back        B2 -> B1 (physical w1, w2);  Xa = B1, Xb = B2
                //   x_fwd_mix     stack Xa -> Xb, launches Xb -> Xa[0, ns) (mix); w2 stays at Xa[ns, 2ns)
                //   x_back_src    Xa[0, ns) -> What at Xb[0, ns), f(t + tau, What) - w2 stack at Xb[ns, 2ns)
                //   x_fwd_corr    Xb[ns, 2ns) -> Xa[0, ns)
                //   x_back_upd    Xa[0, ns) + What -> out (commits the step)
                back2(V, "y_back", 1, 2 * ns, B2, nullptr, B1, UF_STORE);
                double *Xa = B1, *Xb = B2;
                const size_t mix0 = L.size();
                fwd2(V, "x_fwd_mix", 0, 2 * ns, EPI_MIX, Xa, Xb, Xa, false, p.dv(0, 0), p.dv(0, 1));
                for (size_t i = mix0; i < L.size(); ++i)
                    if (L[i].kind == Op::KERNEL) L[i].L.args.mix_w2 = 0;
                back2(V, "x_back_src", 0, ns, Xa, nullptr, Xb, UF_WHAT_SRC, Xa + Fs, Xb + Fs);
                for (int part = 1; part <= 2; ++part) {
                    L.push_back(kernel_op(p.transform(V, part == 1 ? "x_fwd_corr_even" : "x_fwd_corr_odd", 0, false,
                                                      ns, EPI_SCALE, false, Xb + Fs, Xa, false, nullptr, false, part)));
                    L.back().L.args.dA = p.dv(0, 2);
                }
                back2(V, "x_back_upd", 0, ns, Xa, nullptr, out, UF_UPDATE, Xb);
            } else {
            back2(V, "y_back", 1, 2 * ns, B2, B1, B2, UF_STORE);
            double *Xa = B2, *Xb = B1;
            // x_fwd_mix: mix (sigma/delta) -> Xa[0, ns); w2 stays in physical space at Xa[ns, 2ns)
            const size_t mix0 = L.size();
            fwd2(V, "x_fwd_mix", 0, 2 * ns, EPI_MIX, Xa, Xb, Xa, false, p.dv(0, 0), p.dv(0, 1));
            for (size_t i = mix0; i < L.size(); ++i)
                if (L[i].kind == Op::KERNEL) L[i].L.args.mix_w2 = 0;
            // x_back_src: What -> Xa[0, ns); f(t + tau, What) - w2 (stepper.cpp:252) as
            // x_fwd_corr's level-2 stack -> Xb[ns, 2ns)
            back2(V, "x_back_src", 0, ns, Xa, Xb, Xa, UF_WHAT_SRC, Xa + Fs, Xb + Fs);
            for (int part = 1; part <= 2; ++part) {
                L.push_back(kernel_op(p.transform(V, part == 1 ? "x_fwd_corr_even" : "x_fwd_corr_odd", 0, false, ns,
                                                  EPI_SCALE, false, Xb + Fs, Xb, false, nullptr, false, part)));
                L.back().L.args.dA = p.dv(0, 2);
            }
            // x_back_upd: U1 = What + tau Q3(fw) -> out (commits the step)
            back2(V, "x_back_upd", 0, ns, Xb, Xb + Fs, out, UF_UPDATE, Xa);
            }
        } else {
        if (p.dim == 3) {
            L.push_back(kernel_op(p.transform(V, "y_fwd", 1, false, 2 * ns, EPI_SCALE, false, p.W, p.Z)));
            L.back().L.args.dA = p.dv(1, 0);
        } else {
            first_transform(V, 1, const_cast<double*>(in), p.Z, p.W);
        }
        // folded x: y_back also writes the x-reversed W into the idle output state
        // buffer (free until x_back_upd writes U' there, after x_fwd_mix read it)
        double* wrev = p.fold[0] ? out : nullptr;
        L.push_back(kernel_op(p.transform(V, "y_back", 1, true, 2 * ns, EPI_STORE, false, p.Z, p.W)));
        L.back().L.args.out_rev = wrev;
        L.push_back(kernel_op(p.transform(V, "x_fwd_mix", 0, false, 2 * ns, EPI_MIX, false, p.W, p.Z, false, wrev)));
        L.back().L.args.dA = p.dv(0, 0);
        L.back().L.args.dB = p.dv(0, 1);
        L.push_back(kernel_op(p.transform(V, "x_back_src", 0, true, ns, EPI_WHAT_SRC, false, p.Z, p.W)));
        L.push_back(kernel_op(p.transform(V, "x_fwd_corr", 0, false, ns, EPI_CORR, false, p.W + ns * V.F, p.Z)));
        L.back().L.args.aux = p.Z + ns * V.F;
        L.back().L.args.dA = p.dv(0, 2);
        L.push_back(kernel_op(p.transform(V, "x_back_upd", 0, true, ns, EPI_UPDATE, false, p.Z, out)));
        L.back().L.args.aux = p.W;
        }
        if (p.sharded) {
            // global abort agreement, then commit on every rank
            Op fc;
            fc.kind = Op::FAILCODE;
            fc.name = "fail_code";
            L.push_back(fc);
            Op gx;
            gx.kind = Op::EXCHANGE;
            gx.name = "gather_codes";
            for (int s = 0; s < p.G; ++s) {
                gx.sends.push_back({s, p.codes + p.G, sizeof(int)});
                gx.recvs.push_back({s, p.codes + s, sizeof(int)});
            }
            L.push_back(gx);
            Op cm;
            cm.kind = Op::COMMIT;
            cm.name = "commit";
            L.push_back(cm);
        }
    }
    if (p.thomas) ensure_thomas_scratch(p, p.th_need);
    if (p.sharded && !p.local_group) {
        int lo = 0, hi = 0;
        ETD_CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        ETD_CK(cudaStreamCreateWithPriority(&p.xstream, cudaStreamNonBlocking, hi));
        p.sev.resize(2 + 2 * p.zC);
        for (auto& e : p.sev) ETD_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    p.stats.clear();
    for (auto& op : p.steps[0])
        if (op.kind == Op::KERNEL || op.kind == Op::SOURCE || op.kind == Op::THOMAS || op.kind == Op::FOLD ||
            op.kind == Op::UNFOLD || op.kind == Op::ZYFOLD)
            p.stats.push_back({op.L.name, 0, 0, op.L.flops, op.L.bytes, op.L.dense_flops});
    ETD_CK(cudaStreamSynchronize(p.stream));
}

static void launch(const Launch& L, cudaStream_t s) {
    void* args[4] = {const_cast<CUtensorMap*>(&L.tmA), const_cast<CUtensorMap*>(&L.tmB),
                     const_cast<CUtensorMap*>(&L.tmA2), const_cast<ContractArgs*>(&L.args)};
    static const bool one_cta = std::getenv("ETD_ONE_CTA") != nullptr;  // diagnostic: one CTA per SM
    ETD_CK(cudaLaunchKernel(L.k.fn, L.grid, dim3(L.k.threads), args, one_cta ? std::max(L.k.smem, 120000) : L.k.smem, s));
}

// One op of one rank.  EXCHANGE over NCCL here; virtual-rank groups route
// exchanges through group_steps instead.
static void run_op_body(Plan& p, const Op& op, cudaStream_t s);
static void run_op(Plan& p, const Op& op, cudaStream_t s0) {
    const bool ev = p.xstream && !p.local_group;
    const cudaStream_t s = (ev && op.strm == 1) ? p.xstream : s0;
    if (ev && op.wait_ev >= 0) ETD_CK(cudaStreamWaitEvent(s, p.sev[op.wait_ev], 0));
    run_op_body(p, op, s);
    if (ev && op.rec_ev >= 0) ETD_CK(cudaEventRecord(p.sev[op.rec_ev], s));
}

static void run_op_body(Plan& p, const Op& op, cudaStream_t s) {
    switch (op.kind) {
    case Op::NOP: break;
    case Op::KERNEL: launch(op.L, s); break;
    case Op::COPY2D:
        ETD_CK(cudaMemcpy2DAsync(op.dst, op.dpitch, op.src, op.spitch, op.width, op.height,
                                 cudaMemcpyDeviceToDevice, s));
        break;
    case Op::SOURCE: {
        void* args[1] = {const_cast<SourceArgs*>(&op.sargs)};
        ETD_CK(cudaLaunchKernel(op.src_fn, dim3(op.src_blocks), dim3(256), args, 0, s));
        break;
    }
    case Op::THOMAS: {
        void* args[2] = {const_cast<CUtensorMap*>(&op.L.tmA), const_cast<ThomasArgs*>(&op.targs)};
        ETD_CK(cudaLaunchKernel(op.src_fn, dim3(op.src_blocks), dim3(128), args, op.L.k.smem, s));
        break;
    }
    case Op::FOLD: {
        void* args[1] = {const_cast<Fold2Args*>(&op.fargs)};
        ETD_CK(cudaLaunchKernel(reinterpret_cast<const void*>(etd_fold2), dim3(op.src_blocks), dim3(256), args, 0, s));
        break;
    }
    case Op::ZYFOLD: {
        void* args[1] = {const_cast<ZYArgs*>(&op.zargs)};
        ETD_CK(cudaLaunchKernel(reinterpret_cast<const void*>(etd_unfold_fold_zy), dim3(op.src_blocks), dim3(256),
                                args, 0, s));
        break;
    }
    case Op::UNFOLD: {
        void* args[1] = {const_cast<Unfold2Args*>(&op.uargs)};
        ETD_CK(cudaLaunchKernel(op.src_fn, dim3(op.src_blocks), dim3(256), args, 0, s));
        break;
    }
    case Op::FAILCODE: etd_fail_code<<<1, 1, 0, s>>>(p.status, p.codes + p.G); break;
    case Op::COMMIT: etd_commit<<<1, 1, 0, s>>>(p.status, p.codes, p.G, p.tau); break;
    case Op::EXCHANGE: {
        if (p.local_group) throw ConfigError("virtual-rank plans step through etd_group_step");
        auto& nc = Nccl::get();
        // self pieces are device copies; peer pieces one grouped send/recv set
        std::vector<const Piece*> self_s, self_r;
        for (auto& x : op.sends) if (x.peer == p.rank) self_s.push_back(&x);
        for (auto& x : op.recvs) if (x.peer == p.rank) self_r.push_back(&x);
        for (size_t i = 0; i < self_s.size(); ++i)
            ETD_CK(cudaMemcpyAsync(self_r[i]->ptr, self_s[i]->ptr, self_s[i]->bytes, cudaMemcpyDeviceToDevice, s));
        nc.check(nc.GroupStart(), "ncclGroupStart");
        for (auto& x : op.sends)
            if (x.peer != p.rank) nc.check(nc.Send(x.ptr, x.bytes, /*ncclChar*/ 0, x.peer, p.comm, s), "ncclSend");
        for (auto& x : op.recvs)
            if (x.peer != p.rank) nc.check(nc.Recv(x.ptr, x.bytes, /*ncclChar*/ 0, x.peer, p.comm, s), "ncclRecv");
        nc.check(nc.GroupEnd(), "ncclGroupEnd");
        break;
    }
    }
}

static void ensure_graphs(Plan& p) {
    for (int par = 0; par < 2; ++par) {
        if (p.graph[par]) continue;
        cudaGraph_t g;
        ETD_CK(cudaStreamBeginCapture(p.stream, cudaStreamCaptureModeThreadLocal));
        for (auto& op : p.steps[par]) run_op(p, op, p.stream);
        ETD_CK(cudaStreamEndCapture(p.stream, &g));
        ETD_CK(cudaGraphInstantiate(&p.graph[par], g, 0));
        cudaGraphDestroy(g);
    }
}

static void copy_status_from_device(Plan& p) {
    ETD_CK(cudaMemcpyAsync(p.status_host, p.status, sizeof(StepStatus), cudaMemcpyDeviceToHost, p.stream));
    ETD_CK(cudaStreamSynchronize(p.stream));
}

static void reset_status(Plan& p, cudaStream_t s) {
    p.status_host->fail = 0;
    p.status_host->cta_done = 0;
    ETD_CK(cudaMemcpyAsync(p.status, p.status_host, sizeof(StepStatus), cudaMemcpyHostToDevice, s));
}

static void finish_steps(Plan& p, long long n_before) {
    copy_status_from_device(p);
    const long long committed = p.status_host->n - n_before;
    p.cur = (int)((p.cur + committed) & 1);
    if (p.status_host->fail) {
        const int kind = p.status_host->fail;
        const double t = p.status_host->t + ((kind == 2 || kind == 3 || kind == 5) ? p.tau : 0.0);
        if (kind >= 4)  // problems.cpp:126-129: the source throws StepperAbort(t, -1)
            throw AbortError("source domain violation: u >= 1 at t=" + std::to_string(t), t, -1);
        const char* what = kind == 3 ? "step update" : "source";
        throw AbortError(std::string(what) + " produced non-finite values at t=" + std::to_string(t), t,
                         (long)p.status_host->n);
    }
}

static void do_steps(Plan& p, int nsteps) {
    if (nsteps < 0) throw ConfigError("nsteps must be >= 0");
    if (p.local_group) throw ConfigError("virtual-rank plans step through etd_group_step");
    if (nsteps == 0) return;
    copy_status_from_device(p);
    const long long n_before = p.status_host->n;
    reset_status(p, p.stream);
    const bool eager = p.profiling || p.sharded || std::getenv("ETD_DEBUG_CHECKSUM");
    if (eager) {
        // per-kernel device intervals: [event before op, event after op] for KERNEL ops
        std::vector<cudaEvent_t> ev;
        std::vector<std::pair<size_t, size_t>> spans;  // (start ev, stat index)
        auto rec = [&] {
            cudaEvent_t e;
            ETD_CK(cudaEventCreate(&e));
            ETD_CK(cudaEventRecord(e, p.stream));
            ev.push_back(e);
            return ev.size() - 1;
        };
        size_t prev = p.profiling ? rec() : 0;
        const char* dbg = std::getenv("ETD_DEBUG_CHECKSUM");
        unsigned long long* dsum = nullptr;
        if (dbg) ETD_CK(cudaMalloc(&dsum, 16));
        for (int s = 0; s < nsteps; ++s) {
            size_t kidx = 0;
            for (const auto& op : p.steps[(p.cur + s) & 1]) {
                run_op(p, op, p.stream);
                if (dbg && (op.kind == Op::KERNEL || op.kind == Op::SOURCE)) {
                    // checksum every output operand of this op (debugging aid)
                    const double* base = op.kind == Op::SOURCE ? op.sargs.buf : op.L.args.out;
                    const long long F = op.kind == Op::SOURCE ? op.sargs.F : op.L.args.out_stride;
                    const int nout = op.kind == Op::SOURCE ? 2 * p.ns
                                   : op.L.epi == EPI_WHAT_SRC ? 2 * op.L.S
                                   : op.L.epi == EPI_MIX ? op.L.S : op.L.S;
                    for (int o = 0; o < nout; ++o) {
                        unsigned long long h[2];
                        ETD_CK(cudaMemsetAsync(dsum, 0, 16, p.stream));
                        etd_checksum<<<1184, 256, 0, p.stream>>>(base + (size_t)o * F, F, dsum);
                        ETD_CK(cudaMemcpyAsync(h, dsum, 16, cudaMemcpyDeviceToHost, p.stream));
                        ETD_CK(cudaStreamSynchronize(p.stream));
                        std::fprintf(stderr, "ETD_CHECKSUM step %d op %s out %d %016llx %016llx\n", s, op.name.c_str(),
                                     o, h[0], h[1]);
                    }
                }
                if (!p.profiling) continue;
                const size_t e = rec();
                if (op.kind == Op::KERNEL || op.kind == Op::SOURCE || op.kind == Op::THOMAS || op.kind == Op::FOLD ||
                    op.kind == Op::UNFOLD || op.kind == Op::ZYFOLD)
                    spans.push_back({prev, kidx++});
                prev = e;
            }
        }
        ETD_CK(cudaStreamSynchronize(p.stream));
        for (auto& sp : spans) {
            float ms = 0;
            ETD_CK(cudaEventElapsedTime(&ms, ev[sp.first], ev[sp.first + 1]));
            p.stats[sp.second].ms += ms;
            p.stats[sp.second].launches += 1;
        }
        for (auto e : ev) cudaEventDestroy(e);
        if (dsum) cudaFree(dsum);
    } else {
        ensure_graphs(p);
        for (int s = 0; s < nsteps; ++s) ETD_CK(cudaGraphLaunch(p.graph[(p.cur + s) & 1], p.stream));
    }
    ETD_CK(cudaGetLastError());
    finish_steps(p, n_before);
}

// Virtual ranks: G plans of one sharded grid on ONE device, stepped op by op in
// lock-step on the first plan's stream.  No kernel ever waits on another rank;
// an exchange is a set of device copies issued once every rank has finished the
// preceding op.  Exercises the sharded schedule (partition, pack, exchange,
// unpack, global abort agreement) without NCCL or a second GPU.
static void group_steps(std::vector<Plan*>& ps, int nsteps) {
    const int G = (int)ps.size();
    if (G < 1) throw ConfigError("empty group");
    // ETD_SOLO_RANK (timing diagnostic, tools/solo_rank.py): one virtual rank of a G-rank
    // plan runs its own ops with the exchanges skipped (peer data reads as the buffers'
    // zero fill), to time a rank's compute at a G that does not fit one device G times
    const bool solo = G == 1 && ps[0]->local_group && ps[0]->G > 1 && std::getenv("ETD_SOLO_RANK");
    for (int r = 0; r < G; ++r) {
        if (solo) break;
        if (!ps[r]->local_group || ps[r]->G != G || ps[r]->rank != r)
            throw ConfigError("group handles must be virtual ranks 0..G-1 of one sharded plan");
        if (ps[r]->d.device != ps[0]->d.device) throw ConfigError("virtual ranks must share a device");
    }
    if (nsteps < 0) throw ConfigError("nsteps must be >= 0");
    if (nsteps == 0) return;
    for (int r = 1; r < G; ++r)
        for (int par = 0; par < 2; ++par)
            if (ps[r]->steps[par].size() != ps[0]->steps[par].size())
                throw ConfigError("internal: virtual rank " + std::to_string(r) + " has " +
                                  std::to_string(ps[r]->steps[par].size()) + " ops per step, rank 0 has " +
                                  std::to_string(ps[0]->steps[par].size()));
    cudaStream_t s = ps[0]->stream;
    for (auto* p : ps) ETD_CK(cudaStreamSynchronize(p->stream));
    std::vector<long long> before(G);
    for (int r = 0; r < G; ++r) {
        copy_status_from_device(*ps[r]);
        before[r] = ps[r]->status_host->n;
        reset_status(*ps[r], s);
    }
    for (int st = 0; st < nsteps; ++st) {
        const size_t nops = ps[0]->steps[0].size();
        for (size_t k = 0; k < nops; ++k) {
            for (int r = 0; r < G; ++r) {
                Plan& p = *ps[r];
                const Op& op = p.steps[(p.cur + st) & 1][k];
                if (op.kind != Op::EXCHANGE) {
                    run_op(p, op, s);
                    continue;
                }
                if (solo) {
                    // every peer "reports" this rank's own fail code; the data exchanges are skipped
                    if (op.name == "gather_codes")
                        for (size_t i = 0; i < op.sends.size() && i < op.recvs.size(); ++i)
                            ETD_CK(cudaMemcpyAsync(op.recvs[i].ptr, op.sends[i].ptr, op.sends[i].bytes,
                                                   cudaMemcpyDeviceToDevice, s));
                    continue;
                }
                // push this rank's sends into the peers' receive pieces (matched in order)
                std::vector<int> seen(G, 0);
                for (const auto& x : op.sends) {
                    Plan& q = *ps[x.peer];
                    const Op& qo = q.steps[(q.cur + st) & 1][k];
                    int idx = -1, cnt = 0;
                    for (size_t i = 0; i < qo.recvs.size(); ++i)
                        if (qo.recvs[i].peer == r && cnt++ == seen[x.peer]) { idx = (int)i; break; }
                    if (idx < 0 || qo.recvs[idx].bytes != x.bytes)
                        throw CudaError("exchange plan mismatch between virtual ranks");
                    ++seen[x.peer];
                    ETD_CK(cudaMemcpyAsync(qo.recvs[idx].ptr, x.ptr, x.bytes, cudaMemcpyDeviceToDevice, s));
                }
            }
        }
    }
    ETD_CK(cudaGetLastError());
    ETD_CK(cudaStreamSynchronize(s));
    std::string err;
    double et = 0;
    long es = 0;
    for (int r = 0; r < G; ++r) {
        try {
            finish_steps(*ps[r], before[r]);
        } catch (const AbortError& e) {
            err = e.what();
            et = e.t;
            es = e.step;
        }
    }
    if (!err.empty()) throw AbortError(err, et, es);
}

// Host-buffer advance (the reference's value-semantics call shape): unsharded
// plans whose step is source + column (z / y) stages + x stage run it with the
// host<->device copies pipelined against compute (advance_overlapped below); the
// step commit moves to one etd_commit after the chunks.  Everything else takes
// set_state / etd_step / get_state.
// transfer chunks of the pipelined advance; config 4 e2e per chunk count (1 step):
// 6: 745, 8: 727, 12: 713, 16: 714-716, 24: 709, 32: 754, 64: 783 ms
static constexpr int kXferChunks = 16;
static constexpr int kXferChunksMax = 128;
static int xfer_chunks() {  // ETD_XFER_CHUNKS: A/B of the transfer chunk count (default kXferChunks)
    const char* e = std::getenv("ETD_XFER_CHUNKS");
    const int c = e ? std::atoi(e) : kXferChunks;
    return std::max(1, std::min(kXferChunksMax, c));
}

// Index of the first x-stage op.  Everything before it (the source pass and the
// z / y stages) treats x as a batch index, so it can run on x-column ranges.
static int x_stage_index(const Plan& p) {
    const auto& ops = p.steps[0];
    for (size_t k = 0; k < ops.size(); ++k)
        if ((ops[k].kind == Op::KERNEL || ops[k].kind == Op::FOLD || ops[k].kind == Op::UNFOLD) && ops[k].L.mode == 0)
            return (int)k;
    return -1;
}

static bool overlap_eligible(const Plan& p, int nsteps) {
    if (p.sharded || p.profiling || nsteps < 1) return false;
    const auto& ops = p.steps[0];
    const int ix = x_stage_index(p);
    if (ix <= 0 || ops.back().L.name != "x_back_upd") return false;
    for (int k = 0; k < (int)ops.size(); ++k) {
        const Op& op = ops[k];
        if (op.kind != Op::KERNEL && op.kind != Op::SOURCE && op.kind != Op::FOLD && op.kind != Op::UNFOLD &&
            op.kind != Op::ZYFOLD)
            return false;
        if (op.kind != Op::SOURCE && op.L.mode != (k < ix ? 1 : 0)) return false;
        if (op.kind == Op::SOURCE && k >= ix) return false;
    }
    return true;
}

// Host-buffer advance with the copies hidden behind compute:
//  * upload in x-column ranges (strided 2D copies; 55.6 GB/s down to 256-byte row
//    pieces, tools/xfer2d_probe.py).  The first step's source pass and z / y stages
//    run on each range as soon as it lands: they need every y and z of a column but
//    nothing of its neighbours, so ~540 ms of config-4 work covers the ~310 ms upload.
//  * the last step's x stage runs in row chunks (multiples of 128 rows, the largest
//    x-stage tile height); each chunk's rows of U' stream back while the next computes.
//    The y stage is complete before the x stage starts, so a chunk never reads rows
//    a later chunk still has to produce, and x_back_upd's U' (written over the
//    x-reversed W copy in the output state buffer) only lands on rows x_fwd_mix
//    has already consumed.
// Pageable host buffers (a plain std::vector / numpy array, the reference Field's
// storage) cannot be DMA'd asynchronously: a device->host copy into pageable memory
// returns only when it is done, which would serialise the pipeline.  They go
// through a pinned host mirror of the state instead (allocated once per plan):
// host threads copy each upload column range into the mirror just before its H2D
// copy is queued, and copy each downloaded row chunk out of the mirror while the
// next chunk computes.  Pinned (registered) buffers are DMA'd directly.
static bool is_pageable(const void* ptr) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

static int copy_threads() {
    if (const char* e = std::getenv("ETD_COPY_THREADS")) return std::max(1, std::atoi(e));
    return (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
}

// f(lo, hi) over [0, items) split across the host copy threads
template <class F>
static void parallel_rows(long long items, const F& f) {
    const int T = (int)std::max(1LL, std::min<long long>(copy_threads(), items / 64));
    if (T == 1) {
        f(0, items);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(T);
    for (int i = 0; i < T; ++i) th.emplace_back([&, i] { f(items * i / T, items * (i + 1) / T); });
    for (auto& x : th) x.join();
}

static double* ensure_mirror(Plan& p, size_t elems) {
    if (p.mirror_elems < elems) {
        if (p.mirror) ETD_CK(cudaFreeHost(p.mirror));
        p.mirror = nullptr;
        p.mirror_elems = 0;
        ETD_CK(cudaHostAlloc(&p.mirror, elems * sizeof(double), cudaHostAllocDefault));
        p.mirror_elems = elems;
    }
    return p.mirror;
}

static void advance_overlapped(Plan& p, const double* const* hin, double* const* hout, long n, double t,
                               int nsteps) {
    const View& V = p.slab;
    const int ix = x_stage_index(p);
    // column chunk width: a multiple of every column-stage tile height (BM)
    int bm = 32;
    for (int k = 0; k < ix; ++k)
        if (p.steps[0][k].kind == Op::KERNEL) bm = std::max(bm, p.steps[0][k].L.k.bm);
    // Column ranges of the upload.  The column phase ends at about max(upload,
    // first range's upload + column compute) + the last range's compute, and wider
    // ranges upload faster (2D copies of (x1-x0)*8-byte row pieces, config 4 with
    // compute running: 48.4 GB/s at 512 B, 51.7 at 1 KB, 53.5 at 2 KB,
    // tools/e2e_timeline.py).  So: one narrow range first (compute starts early),
    // wide ranges in the middle, narrowing ranges at the end (short tail).
    // ETD_XFER_CHUNKS=N restores N uniform ranges (A/B).
    std::vector<int> colb{0};
    const int NX = xfer_chunks();
    if (std::getenv("ETD_XFER_CHUNKS") || V.nx < 16 * bm) {
        const int XW = round_up((V.nx + NX - 1) / NX, bm);
        for (int x = XW; x < V.nx; x += XW) colb.push_back(x);
    } else {
        const int base = round_up((V.nx + 7) / 8, bm);
        const int tail[3] = {3 * bm, 2 * bm, bm};
        int x = bm;
        colb.push_back(x);
        const int mid_end = (V.nx - (tail[0] + tail[1] + tail[2])) / bm * bm;  // range starts stay tile aligned
        while (x + base < mid_end) colb.push_back(x += base);
        if (mid_end > x) colb.push_back(x = mid_end);
        for (int t : tail)
            if (x + t < V.nx) colb.push_back(x += t);
    }
    colb.push_back(V.nx);
    const int CX = (int)colb.size() - 1;
    const long long R = (long long)V.ny * V.nz;
    const int C = (int)std::max(1LL, std::min<long long>(NX, R / 128));
    if (CX > kXferChunksMax) throw ConfigError("internal: too many upload ranges");
    if (!p.cstream) {
        ETD_CK(cudaStreamCreateWithFlags(&p.cstream, cudaStreamNonBlocking));
        p.xev.resize(3 * kXferChunksMax + 1);
        for (auto& e : p.xev) ETD_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    cudaEvent_t* ev_in = p.xev.data();
    cudaEvent_t* ev_out = p.xev.data() + kXferChunksMax;
    cudaEvent_t* ev_dl = p.xev.data() + 2 * kXferChunksMax;  // download of row chunk c landed
    cudaEvent_t ev_start = p.xev[3 * kXferChunksMax];
    // pageable buffers go through the pinned mirror [species][R][nx] (host layout)
    const size_t cnt = (size_t)R * V.nx;
    bool pg_in[2] = {false, false}, pg_out[2] = {false, false}, any_in = false, any_out = false;
    for (int sp = 0; sp < p.ns; ++sp) {
        pg_in[sp] = is_pageable(hin[sp]);
        pg_out[sp] = is_pageable(hout[sp]);
        any_in |= pg_in[sp];
        any_out |= pg_out[sp];
    }
    double* mir = (any_in || any_out) ? ensure_mirror(p, cnt * p.ns) : nullptr;
    // pageable outputs are typically fresh allocations (a new Field / numpy array per
    // call): ask for transparent huge pages before the copy threads first-touch them
    for (int sp = 0; sp < p.ns && any_out; ++sp) {
        if (!pg_out[sp]) continue;
        const uintptr_t a = reinterpret_cast<uintptr_t>(hout[sp]), pg = 2u << 20;
        const uintptr_t lo = (a + pg - 1) / pg * pg, hi = (a + cnt * 8) / pg * pg;
        if (hi > lo) madvise(reinterpret_cast<void*>(lo), hi - lo, MADV_HUGEPAGE);
    }
    p.status_host->n = n;
    p.status_host->t = t;
    p.status_host->fail = 0;
    p.status_host->cta_done = 0;
    ETD_CK(cudaMemcpyAsync(p.status, p.status_host, sizeof(StepStatus), cudaMemcpyHostToDevice, p.stream));
    ETD_CK(cudaEventRecord(ev_start, p.stream));
    ETD_CK(cudaStreamWaitEvent(p.cstream, ev_start, 0));
    // x-stage row chunks (multiples of 128 rows): a small first chunk so the
    // download starts early, then uniform chunks (the download, not the x stage,
    // paces the rest)
    const long long R1 = C > 1 ? std::max<long long>(128, R / (4LL * C) / 128 * 128) : R;
    auto rowb = [&](int c) -> long long {
        if (c <= 0) return 0;
        if (c >= C) return R;
        return R1 + (R - R1) * (c - 1) / (C - 1) / 128 * 128;
    };
    double* st_in = p.state[p.cur];
    auto upload = [&](int c) {
        const int x0 = colb[c], x1 = colb[c + 1];
        for (int sp = 0; sp < p.ns; ++sp) {
            const double* src = hin[sp];
            if (pg_in[sp]) {
                double* m = mir + (size_t)sp * cnt;
                const double* h = hin[sp];
                parallel_rows(R, [&](long long r0, long long r1) {
                    for (long long r = r0; r < r1; ++r)
                        std::memcpy(m + r * V.nx + x0, h + r * V.nx + x0, (size_t)(x1 - x0) * 8);
                });
                src = m;
            }
            ETD_CK(cudaMemcpy2DAsync(st_in + (size_t)sp * V.F + x0, (size_t)V.pitch * 8, src + x0,
                                     (size_t)V.nx * 8, (size_t)(x1 - x0) * 8, (size_t)R, cudaMemcpyHostToDevice,
                                     p.cstream));
        }
        ETD_CK(cudaEventRecord(ev_in[c], p.cstream));
    };
    // pinned inputs: every column range is queued up front; pageable ones are
    // staged range by range inside the first step's column loop, so each range's
    // compute is queued right behind its copy while the host stages the next
    if (!any_in)
        for (int c = 0; c < CX; ++c) upload(c);
    // ETD_TIMELINE: device timestamps of the pipeline (uploads, column chunks, x
    // chunks, downloads) printed to stderr after the call (measurement aid)
    const bool tl = std::getenv("ETD_TIMELINE") != nullptr;
    std::vector<std::pair<std::string, cudaEvent_t>> tev;
    auto mark = [&](const std::string& what, cudaStream_t st) {
        if (!tl) return;
        cudaEvent_t e;
        ETD_CK(cudaEventCreate(&e));
        ETD_CK(cudaEventRecord(e, st));
        tev.push_back({what, e});
    };
    mark("start", p.stream);
    if (tl && !any_in)
        for (int c = 0; c < CX; ++c) {
            ETD_CK(cudaStreamWaitEvent(p.cstream, ev_in[c], 0));
            mark("up" + std::to_string(c), p.cstream);
        }
    for (int s = 0; s < nsteps; ++s) {
        const auto& ops = p.steps[(p.cur + s) & 1];
        const bool first = s == 0, last = s == nsteps - 1;
        // source + z / y stages: per x-column range in the first step
        if (first) {
            for (int c = 0; c < CX; ++c) {
                if (any_in) upload(c);
                if (c > 0) mark("col" + std::to_string(c - 1), p.stream);
                ETD_CK(cudaStreamWaitEvent(p.stream, ev_in[c], 0));
                const int x0 = colb[c], x1 = colb[c + 1];
                for (int k = 0; k < ix; ++k) {
                    if (ops[k].kind == Op::SOURCE) {
                        Op o = ops[k];
                        o.sargs.x0 = x0;
                        o.sargs.x1 = x1;
                        run_op(p, o, p.stream);
                    } else if (ops[k].kind == Op::FOLD) {
                        Op o = ops[k];
                        o.fargs.x0 = x0;
                        o.fargs.x1 = x1;
                        run_op(p, o, p.stream);
                    } else if (ops[k].kind == Op::UNFOLD) {
                        Op o = ops[k];
                        o.uargs.x0 = x0;
                        o.uargs.x1 = x1;
                        run_op(p, o, p.stream);
                    } else if (ops[k].kind == Op::ZYFOLD) {
                        Op o = ops[k];
                        o.zargs.x0 = x0;
                        o.zargs.x1 = x1;
                        run_op(p, o, p.stream);
                    } else {
                        Launch L = ops[k].L;
                        L.args.mtile0 = x0 / L.k.bm;
                        L.grid.y = (unsigned)((x1 + L.k.bm - 1) / L.k.bm - x0 / L.k.bm);
                        launch(L, p.stream);
                    }
                }
            }
        } else {
            for (int k = 0; k < ix; ++k) run_op(p, ops[k], p.stream);
        }
        if (first) mark("col" + std::to_string(CX - 1), p.stream);
        // x stage
        if (!last) {
            for (size_t k = ix; k < ops.size(); ++k) run_op(p, ops[k], p.stream);
            continue;
        }
        const Op& upd = ops.back();
        // pageable outputs: copy row chunk c out of the mirror once its download landed
        auto drain = [&](int c) {
            const long long r0 = rowb(c), r1 = rowb(c + 1);
            if (!any_out || r1 <= r0) return;
            ETD_CK(cudaEventSynchronize(ev_dl[c]));
            for (int sp = 0; sp < p.ns; ++sp) {
                if (!pg_out[sp]) continue;
                const double* m = mir + (size_t)sp * cnt + r0 * V.nx;
                double* h = hout[sp] + r0 * V.nx;
                parallel_rows(r1 - r0, [&](long long a, long long b) {
                    std::memcpy(h + a * V.nx, m + a * V.nx, (size_t)(b - a) * V.nx * 8);
                });
            }
        };
        int prev = -1;  // last queued row chunk whose pageable copy-out is pending
        for (int c = 0; c < C; ++c) {
            const long long r0 = rowb(c), r1 = rowb(c + 1);
            if (r1 <= r0) continue;
            for (size_t k = ix; k < ops.size(); ++k) {
                if (ops[k].kind == Op::FOLD) {
                    Op o = ops[k];
                    o.fargs.r0 = r0;
                    o.fargs.r1 = r1;
                    run_op(p, o, p.stream);
                    continue;
                }
                if (ops[k].kind == Op::UNFOLD) {
                    Op o = ops[k];
                    o.uargs.r0 = r0;
                    o.uargs.r1 = r1;
                    o.uargs.commit = 0;
                    run_op(p, o, p.stream);
                    continue;
                }
                Launch L = ops[k].L;
                L.args.mtile0 = (int)(r0 / L.k.bm);
                L.grid.y = (unsigned)((r1 + L.k.bm - 1) / L.k.bm - r0 / L.k.bm);
                L.args.commit = 0;
                launch(L, p.stream);
            }
            ETD_CK(cudaEventRecord(ev_out[c], p.stream));
            mark("x" + std::to_string(c), p.stream);
            ETD_CK(cudaStreamWaitEvent(p.cstream, ev_out[c], 0));
            for (int sp = 0; sp < p.ns; ++sp)
                ETD_CK(cudaMemcpy2DAsync((pg_out[sp] ? mir + (size_t)sp * cnt : hout[sp]) + r0 * V.nx,
                                         (size_t)V.nx * 8, upd.L.args.out + (size_t)sp * V.F + r0 * V.pitch,
                                         (size_t)V.pitch * 8, (size_t)V.nx * 8, (size_t)(r1 - r0),
                                         cudaMemcpyDeviceToHost, p.cstream));
            ETD_CK(cudaEventRecord(ev_dl[c], p.cstream));
            mark("down" + std::to_string(c), p.cstream);
            if (prev >= 0) drain(prev);
            prev = c;
        }
        etd_commit<<<1, 1, 0, p.stream>>>(p.status, nullptr, 0, p.tau);
        if (prev >= 0) drain(prev);
    }
    ETD_CK(cudaGetLastError());
    ETD_CK(cudaStreamSynchronize(p.cstream));
    if (tl) {
        ETD_CK(cudaDeviceSynchronize());
        for (auto& [what, e] : tev) {
            float ms = 0;
            ETD_CK(cudaEventElapsedTime(&ms, tev[0].second, e));
            std::fprintf(stderr, "ETD_TIMELINE %s %.3f\n", what.c_str(), ms);
        }
        for (auto& te : tev) cudaEventDestroy(te.second);
    }
    finish_steps(p, n);
}

static void set_state(Plan& p, int species, const double* host, size_t count, long n, double t) {
    if (species < 0 || species >= p.ns) throw ConfigError("species index out of range");
    const View& v = p.slab;
    if (count != (size_t)v.nx * v.ny * v.nz) throw ConfigError("state shape does not match plan grid");
    double* dst = p.state[p.cur] + (size_t)species * v.F;
    ETD_CK(cudaMemcpy2DAsync(dst, v.pitch * 8, host, (size_t)v.nx * 8, (size_t)v.nx * 8, (size_t)v.ny * v.nz,
                             cudaMemcpyHostToDevice, p.stream));
    p.status_host->n = n;
    p.status_host->t = t;
    p.status_host->fail = 0;
    p.status_host->cta_done = 0;
    ETD_CK(cudaMemcpyAsync(p.status, p.status_host, sizeof(StepStatus), cudaMemcpyHostToDevice, p.stream));
    ETD_CK(cudaStreamSynchronize(p.stream));
}

static void get_state(Plan& p, int species, double* host, size_t count, long* n, double* t) {
    if (species < 0 || species >= p.ns) throw ConfigError("species index out of range");
    const View& v = p.slab;
    if (count != (size_t)v.nx * v.ny * v.nz) throw ConfigError("output shape does not match plan grid");
    const double* src = p.state[p.cur] + (size_t)species * v.F;
    ETD_CK(cudaMemcpy2DAsync(host, (size_t)v.nx * 8, src, v.pitch * 8, (size_t)v.nx * 8, (size_t)v.ny * v.nz,
                             cudaMemcpyDeviceToHost, p.stream));
    copy_status_from_device(p);
    if (n) *n = (long)p.status_host->n;
    if (t) *t = p.status_host->t;
}

// ---- ETRD snapshots (reference field.cpp:32-81): "ETRD", u32 version 1, u32 dim,
// u32 shape[3], f64 time, nx*ny*nz f64 (x-fastest).  Streamed through a pinned
// staging buffer so a multi-GB field never needs a full host copy.  Sharded plans
// write/read their own z-slab (shape nx, ny, z1-z0).
static bool field_finite(Plan& p, const double* f) {
    int* flag = p.codes ? p.codes : nullptr;
    int* tmp = nullptr;
    if (!flag) {
        ETD_CK(cudaMalloc(&tmp, sizeof(int)));
        flag = tmp;
    }
    ETD_CK(cudaMemsetAsync(flag, 0, sizeof(int), p.stream));
    etd_nonfinite_scan<<<148 * 8, 256, 0, p.stream>>>(f, p.slab.F, flag);
    int h = 0;
    ETD_CK(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, p.stream));
    ETD_CK(cudaStreamSynchronize(p.stream));
    if (tmp) cudaFree(tmp);
    return h == 0;
}

struct PinnedBuf {
    double* ptr = nullptr;
    size_t elems = 0;
    explicit PinnedBuf(size_t n) : elems(n) { ETD_CK(cudaMallocHost(&ptr, n * sizeof(double))); }
    ~PinnedBuf() { if (ptr) cudaFreeHost(ptr); }
};

static void save_snapshot(Plan& p, int species, const char* path) {
    if (species < 0 || species >= p.ns) throw ConfigError("species index out of range");
    const View& v = p.slab;
    const double* src = p.state[p.cur] + (size_t)species * v.F;
    if (!field_finite(p, src)) throw NumericsError("refusing to save field with non-finite entries");
    copy_status_from_device(p);
    FILE* fp = std::fopen(path, "wb");
    if (!fp) throw ConfigError(std::string("cannot open ") + path + " for writing");
    std::unique_ptr<FILE, int (*)(FILE*)> guard(fp, &std::fclose);
    const uint32_t hdr[5] = {1u, (uint32_t)p.dim, (uint32_t)v.nx, (uint32_t)v.ny, (uint32_t)(p.dim == 3 ? v.nz : 1)};
    const double t = p.status_host->t;
    bool ok = std::fwrite("ETRD", 1, 4, fp) == 4 && std::fwrite(hdr, 4, 5, fp) == 5 && std::fwrite(&t, 8, 1, fp) == 1;
    const size_t rows = (size_t)v.ny * v.nz, per = std::max<size_t>(1, (32u << 20) / v.nx);
    PinnedBuf buf(per * v.nx);
    for (size_t r0 = 0; ok && r0 < rows; r0 += per) {
        const size_t nr = std::min(per, rows - r0);
        ETD_CK(cudaMemcpy2DAsync(buf.ptr, (size_t)v.nx * 8, src + r0 * v.pitch, v.pitch * 8, (size_t)v.nx * 8, nr,
                                 cudaMemcpyDeviceToHost, p.stream));
        ETD_CK(cudaStreamSynchronize(p.stream));
        ok = std::fwrite(buf.ptr, 8, nr * v.nx, fp) == nr * v.nx;
    }
    if (!ok) throw ConfigError(std::string("short write to ") + path);
}

static void load_snapshot(Plan& p, int species, const char* path, long n) {
    if (species < 0 || species >= p.ns) throw ConfigError("species index out of range");
    const View& v = p.slab;
    FILE* fp = std::fopen(path, "rb");
    if (!fp) throw ConfigError(std::string("cannot open ") + path);
    std::unique_ptr<FILE, int (*)(FILE*)> guard(fp, &std::fclose);
    char magic[4];
    uint32_t hdr[5];
    double t = 0.0;
    if (std::fread(magic, 1, 4, fp) != 4 || std::memcmp(magic, "ETRD", 4) != 0)
        throw ConfigError(std::string(path) + ": not a field snapshot");
    if (std::fread(hdr, 4, 5, fp) != 5 || hdr[0] != 1u) throw ConfigError(std::string(path) + ": unsupported version");
    if ((int)hdr[1] != p.dim || (int)hdr[2] != v.nx || (int)hdr[3] != v.ny ||
        (int)hdr[4] != (p.dim == 3 ? v.nz : 1))
        throw ConfigError(std::string(path) + ": snapshot shape does not match plan grid");
    if (std::fread(&t, 8, 1, fp) != 1) throw ConfigError(std::string(path) + ": truncated snapshot");
    // staged in the step scratch (free between steps; pads zero like the state's), so a
    // truncated or non-finite file leaves the live state untouched (the reference's
    // load_field has no side effects on failure, field.cpp:59-81)
    double* stage = p.Z;
    const size_t rows = (size_t)v.ny * v.nz, per = std::max<size_t>(1, (32u << 20) / v.nx);
    PinnedBuf buf(per * v.nx);
    ETD_CK(cudaMemsetAsync(stage, 0, (size_t)v.F * 8, p.stream));
    for (size_t r0 = 0; r0 < rows; r0 += per) {
        const size_t nr = std::min(per, rows - r0);
        if (std::fread(buf.ptr, 8, nr * v.nx, fp) != nr * v.nx)
            throw ConfigError(std::string(path) + ": truncated snapshot");
        ETD_CK(cudaMemcpy2DAsync(stage + r0 * v.pitch, v.pitch * 8, buf.ptr, (size_t)v.nx * 8, (size_t)v.nx * 8, nr,
                                 cudaMemcpyHostToDevice, p.stream));
        ETD_CK(cudaStreamSynchronize(p.stream));
    }
    if (!field_finite(p, stage)) throw NumericsError(std::string(path) + ": snapshot has non-finite entries");
    double* dst = p.state[p.cur] + (size_t)species * v.F;
    ETD_CK(cudaMemcpyAsync(dst, stage, (size_t)v.F * 8, cudaMemcpyDeviceToDevice, p.stream));
    // a snapshot carries t only; restart at n = round(t / tau) unless given
    p.status_host->n = n >= 0 ? n : (long long)std::llround(t / p.tau);
    p.status_host->t = t;
    p.status_host->fail = 0;
    p.status_host->cta_done = 0;
    ETD_CK(cudaMemcpyAsync(p.status, p.status_host, sizeof(StepStatus), cudaMemcpyHostToDevice, p.stream));
    ETD_CK(cudaStreamSynchronize(p.stream));
}

static void debug_transform(Plan& p, int species, int axis, int back, int ell, int apply_q,
                            const double* in, double* out) {
    if (axis < 0 || axis >= p.dim) throw ConfigError("axis out of range for field dimension");
    if (p.sharded) throw ConfigError("debug transforms run on unsharded plans");
    if (species < 0 || species >= p.ns) throw ConfigError("species index out of range");
    if (ell < 0 || ell > 3) throw ConfigError("ell must be 1, 2, or 3");
    const View& v = p.slab;
    ETD_CK(cudaMemcpy2DAsync(p.W, v.pitch * 8, in, (size_t)v.nx * 8, (size_t)v.nx * 8, (size_t)v.ny * v.nz,
                             cudaMemcpyHostToDevice, p.stream));
    reset_status(p, p.stream);
    const double* result = nullptr;
    if (p.thomas) {
        // apply_Q_thomas (thomas.cpp:128-160) of field `species`
        if (!apply_q || ell < 1) throw ConfigError("Thomas plans support only apply_q with ell in 1..3");
        ETD_CK(cudaMemcpyAsync(p.W + (size_t)species * v.F, p.W, (size_t)v.F * 8, cudaMemcpyDeviceToDevice,
                               p.stream));
        Op o = p.thomas_op("dbg_thomas", axis, TH_STORE, p.W, p.Z, 1, ell, species);
        ensure_thomas_scratch(p, p.th_need);
        o.targs.scratch = p.thscr;
        run_op(p, o, p.stream);
        result = p.Z + (size_t)species * v.F;
    } else if (apply_q) {
        if (ell < 1) throw ConfigError("apply_q needs ell in 1..3");
        // folded x: the forward reads its mirror from a host-reversed copy (FOLD 3)
        double* rev = nullptr;
        if (p.fold2[axis]) {
            // second-level split: stack -> even/odd-mode launches -> backward
            double* tmp = p.state[1 - p.cur];
            run_op(p, p.fold_op(v, "dbg_fold", axis, p.W, tmp, 1), p.stream);
            for (int part = 1; part <= 2; ++part) {
                Launch f = p.transform(v, "dbg_fwd", axis, false, 1, EPI_SCALE, false, tmp, p.Z, false, nullptr,
                                       false, part);
                f.args.dA = p.dv(axis, 6 + ell - 1) + species * p.dmax;
                launch(f, p.stream);
            }
            if (p.back6) {
                launch(p.transform(v, "dbg_back", axis, true, 1, EPI_STORE, false, p.Z, p.W + v.F, false, nullptr,
                                   false, 6),
                       p.stream);
            } else {
                for (int part = 3; part <= 4; ++part)
                    launch(p.transform(v, "dbg_back", axis, true, 1, EPI_STORE, false, p.Z, tmp, false, nullptr, false,
                                       part),
                           p.stream);
                run_op(p, p.unfold_op(v, "dbg_unfold", axis, UF_STORE, tmp, p.W + v.F, 1), p.stream);
            }
            result = p.W + v.F;
        } else {
        if (axis == 0 && p.fold[0]) {
            std::vector<double> hr((size_t)v.nx * v.ny * v.nz);
            for (size_t r = 0; r < (size_t)v.ny * v.nz; ++r)
                for (int i = 0; i < v.nx; ++i) hr[r * v.nx + i] = in[r * v.nx + (v.nx - 1 - i)];
            rev = p.state[1 - p.cur];
            ETD_CK(cudaMemcpy2DAsync(rev, v.pitch * 8, hr.data(), (size_t)v.nx * 8, (size_t)v.nx * 8,
                                     (size_t)v.ny * v.nz, cudaMemcpyHostToDevice, p.stream));
            ETD_CK(cudaStreamSynchronize(p.stream));
        }
        Launch f = p.transform(v, "dbg_fwd", axis, false, 1, EPI_SCALE, false, p.W, p.Z, false, rev);
        f.args.dA = p.dv(axis, 6 + ell - 1) + species * p.dmax;
        Launch b = p.transform(v, "dbg_back", axis, true, 1, EPI_STORE, false, p.Z, p.W + v.F);
        launch(f, p.stream);
        launch(b, p.stream);
        result = p.W + v.F;
        }
    } else {
        // one direction in natural mode order: the dense kernel
        Launch f = p.transform(v, "dbg", axis, back != 0, 1, ell ? EPI_SCALE : EPI_STORE, false, p.W, p.Z, true);
        if (ell) f.args.dA = p.dvn(axis, 3 + ell - 1, 0) + species * p.dmax;
        launch(f, p.stream);
        result = p.Z;
    }
    ETD_CK(cudaGetLastError());
    ETD_CK(cudaMemcpy2DAsync(out, (size_t)v.nx * 8, result, v.pitch * 8, (size_t)v.nx * 8, (size_t)v.ny * v.nz,
                             cudaMemcpyDeviceToHost, p.stream));
    ETD_CK(cudaStreamSynchronize(p.stream));
}

}  // namespace etd

// =================================================================== C-ABI
using etd::CudaError;  // for ETD_CK in the C-ABI shims

struct etd_handle {
    std::unique_ptr<etd::Plan> plan;
    std::string msg;
    double t = 0;
    long step = 0;
};

namespace {
thread_local std::string g_create_error;

template <class F>
int guarded(etd_handle* h, F&& f) {
    try {
        f();
        if (h) h->msg.clear();
        return ETD_OK;
    } catch (const etd::AbortError& e) {
        if (h) { h->msg = e.what(); h->t = e.t; h->step = e.step; }
        return ETD_ERR_ABORT;
    } catch (const etd::ConfigError& e) {
        if (h) h->msg = e.what(); else g_create_error = e.what();
        return ETD_ERR_CONFIG;
    } catch (const etd::NumericsError& e) {
        if (h) h->msg = e.what(); else g_create_error = e.what();
        return ETD_ERR_NUMERICS;
    } catch (const etd::NoDevice& e) {
        if (h) h->msg = e.what(); else g_create_error = e.what();
        return ETD_ERR_NODEVICE;
    } catch (const etd::MemoryGuardError& e) {
        if (h) h->msg = e.what(); else g_create_error = e.what();
        return ETD_ERR_MEMORY;
    } catch (const std::bad_alloc& e) {
        if (h) h->msg = "host allocation failed"; else g_create_error = "host allocation failed";
        return ETD_ERR_MEMORY;
    } catch (const std::exception& e) {
        if (h) h->msg = e.what(); else g_create_error = e.what();
        cudaGetLastError();  // a non-sticky launch/API error must not surface in the next call
        return ETD_ERR_CUDA;
    }
}
}  // namespace

extern "C" {

double etd_setup_phi(int which, double x) {
    return which == 1 ? etd::phi1(x) : which == 2 ? etd::phi2(x) : std::nan("");
}

int etd_abi_version(void) { return ETD_B200_ABI_VERSION; }

int etd_create(const etd_desc* desc, etd_handle** out) {
    if (!desc || !out) return ETD_ERR_CONFIG;
    *out = nullptr;
    auto h = std::make_unique<etd_handle>();
    h->plan = std::make_unique<etd::Plan>();
    g_create_error.clear();
    int rc = guarded(nullptr, [&] { etd::build_plan(*h->plan, *desc); });
    if (rc != ETD_OK) {
        // keep the message reachable through etd_last_error(NULL, ...)
        return rc;
    }
    *out = h.release();
    return ETD_OK;
}

int etd_plan_device_bytes(const etd_desc* desc, unsigned long long* bytes) {
    return guarded(nullptr, [&] {
        if (!desc || !bytes) throw etd::ConfigError("null argument");
        etd::validate(*desc);
        *bytes = etd::plan_device_bytes(*desc);
    });
}

int etd_destroy(etd_handle* h) {
    delete h;
    return ETD_OK;
}

int etd_slab_range(const etd_handle* h, int* z0, int* z1) {
    if (!h) return ETD_ERR_CONFIG;
    const auto& p = *h->plan;
    if (z0) *z0 = p.dim == 3 ? p.zlo[p.rank] : 0;
    if (z1) *z1 = p.dim == 3 ? p.zhi[p.rank] : 1;
    return ETD_OK;
}

int etd_zslab_partition(int n, int world_size, int rank, int* lo, int* hi) {
    if (n < 1 || world_size < 1 || rank < 0 || rank >= world_size || world_size > n || !lo || !hi)
        return ETD_ERR_CONFIG;
    etd::partition(n, world_size, rank, *lo, *hi);
    return ETD_OK;
}

int etd_sharded_schedule(int nx, int ny, int nz, int nspecies, int world_size, int rank, long long pitch,
                         int chunks, long long* out, int capacity, int* count) {
    if (!count || world_size < 1 || rank < 0 || rank >= world_size || world_size > nz || world_size > ny ||
        nspecies < 1 || nspecies > 2 || pitch < nx || chunks < 1)
        return ETD_ERR_CONFIG;
    const auto recs = etd::sharded_schedule(nx, ny, nz, nspecies, world_size, rank, pitch, chunks);
    *count = (int)recs.size();
    if (out) {
        if (capacity < (int)recs.size()) return ETD_ERR_CONFIG;
        std::memcpy(out, recs.data(), recs.size() * sizeof(etd::SchedRec));
    }
    return ETD_OK;
}

int etd_sharded_recv_rows(int ny, int nz, int nspecies, int world_size, int rank, long long pitch, int chunks,
                          long long* out) {
    if (!out || world_size < 1 || rank < 0 || rank >= world_size || world_size > nz || world_size > ny ||
        nspecies < 1 || nspecies > 2 || chunks < 1)
        return ETD_ERR_CONFIG;
    const auto t = etd::recv_row_table(ny, nz, nspecies, world_size, rank, pitch, chunks);
    std::memcpy(out, t.data(), t.size() * sizeof(long long));
    return ETD_OK;
}

int etd_nccl_unique_id(void* out) {
    if (!out) return ETD_ERR_CONFIG;
    return guarded(nullptr, [&] {
        auto& nc = etd::Nccl::get();
        ncclUniqueId id;
        nc.check(nc.GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(out, &id, sizeof(id));
    });
}

int etd_group_step(etd_handle** hs, int count, int nsteps) {
    if (!hs || count < 1) return ETD_ERR_CONFIG;
    std::vector<etd::Plan*> ps;
    for (int i = 0; i < count; ++i) {
        if (!hs[i]) return ETD_ERR_CONFIG;
        ps.push_back(hs[i]->plan.get());
    }
    return guarded(hs[0], [&] { etd::group_steps(ps, nsteps); });
}

int etd_set_state(etd_handle* h, int species, const double* host, size_t count, long n, double t) {
    if (!h || !host) return ETD_ERR_CONFIG;
    return guarded(h, [&] { etd::set_state(*h->plan, species, host, count, n, t); });
}

int etd_get_state(etd_handle* h, int species, double* host, size_t count, long* n, double* t) {
    if (!h || !host) return ETD_ERR_CONFIG;
    return guarded(h, [&] { etd::get_state(*h->plan, species, host, count, n, t); });
}

int etd_step(etd_handle* h, int nsteps) {
    if (!h) return ETD_ERR_CONFIG;
    return guarded(h, [&] { etd::do_steps(*h->plan, nsteps); });
}

int etd_advance(etd_handle* h, const double* u, const double* v, long n, double t, int nsteps, double* u_out,
                double* v_out, long* n_out, double* t_out) {
    if (!h || !u || !u_out) return ETD_ERR_CONFIG;
    auto& p = *h->plan;
    if (p.ns == 2 && (!v || !v_out)) return ETD_ERR_CONFIG;
    const size_t cnt = (size_t)p.slab.nx * p.slab.ny * p.slab.nz;
    if (etd::overlap_eligible(p, nsteps)) {
        const double* hin[2] = {u, v};
        double* hout[2] = {u_out, v_out};
        int rs = guarded(h, [&] { etd::advance_overlapped(p, hin, hout, n, t, nsteps); });
        if (rs == ETD_OK) {
            if (n_out) *n_out = (long)p.status_host->n;
            if (t_out) *t_out = p.status_host->t;
            return ETD_OK;
        }
        if (rs != ETD_ERR_ABORT) return rs;
        // abort: hand back the last good state (the input of the failing step)
        std::string keep = h->msg;
        double kt = h->t;
        long ks = h->step;
        guarded(h, [&] {
            etd::get_state(p, 0, u_out, cnt, n_out, t_out);
            if (p.ns == 2) etd::get_state(p, 1, v_out, cnt, n_out, t_out);
        });
        h->msg = keep; h->t = kt; h->step = ks;
        return rs;
    }
    int rc = guarded(h, [&] {
        etd::set_state(p, 0, u, cnt, n, t);
        if (p.ns == 2) etd::set_state(p, 1, v, cnt, n, t);
    });
    if (rc) return rc;
    int rs = etd_step(h, nsteps);
    std::string keep = h->msg;
    double kt = h->t;
    long ks = h->step;
    rc = guarded(h, [&] {
        etd::get_state(p, 0, u_out, cnt, n_out, t_out);
        if (p.ns == 2) etd::get_state(p, 1, v_out, cnt, n_out, t_out);
    });
    if (rs) { h->msg = keep; h->t = kt; h->step = ks; return rs; }
    return rc;
}

int etd_last_error(const etd_handle* h, char* msg, size_t len, double* t, long* step) {
    const std::string& m = h ? h->msg : g_create_error;
    if (msg && len) {
        std::strncpy(msg, m.c_str(), len - 1);
        msg[len - 1] = 0;
    }
    if (t) *t = h ? h->t : 0.0;
    if (step) *step = h ? h->step : 0;
    return ETD_OK;
}

unsigned long long etd_stream(const etd_handle* h) {
    return h ? reinterpret_cast<unsigned long long>(h->plan->stream) : 0ull;
}

int etd_comm_ranks(const etd_handle* h, int* out) {
    return guarded(const_cast<etd_handle*>(h), [&] {
        if (!h || !out) throw etd::ConfigError("null argument");
        const etd::Plan& p = *h->plan;
        *out = p.G;
        if (p.sharded && !p.local_group) {
            auto& nc = etd::Nccl::get();
            nc.check(nc.CommCount(p.comm, out), "ncclCommCount");
        }
    });
}

int etd_launches_per_step(const etd_handle* h) {
    if (!h) return 0;
    int k = 0;
    for (const auto& op : h->plan->steps[0]) k += op.kind != etd::Op::COPY2D && op.kind != etd::Op::EXCHANGE;
    return k;
}

int etd_set_profiling(etd_handle* h, int on) {
    if (!h) return ETD_ERR_CONFIG;
    h->plan->profiling = on != 0;
    for (auto& s : h->plan->stats) { s.ms = 0; s.launches = 0; }
    return ETD_OK;
}

int etd_stage_count(const etd_handle* h) { return h ? (int)h->plan->stats.size() : 0; }

int etd_stage_info(const etd_handle* h, int i, char* name, size_t len, double* ms_total, long* launches,
                   double* flops, double* bytes) {
    if (!h || i < 0 || i >= (int)h->plan->stats.size()) return ETD_ERR_CONFIG;
    const auto& s = h->plan->stats[i];
    if (name && len) {
        std::strncpy(name, s.name.c_str(), len - 1);
        name[len - 1] = 0;
    }
    if (ms_total) *ms_total = s.ms;
    if (launches) *launches = s.launches;
    if (flops) *flops = s.flops;
    if (bytes) *bytes = s.bytes;
    return ETD_OK;
}

int etd_stage_flops(const etd_handle* h, int i, double* executed, double* dense) {
    if (!h || i < 0 || i >= (int)h->plan->stats.size()) return ETD_ERR_CONFIG;
    const auto& s = h->plan->stats[i];
    if (executed) *executed = s.flops;
    if (dense) *dense = s.dense_flops > 0 ? s.dense_flops : s.flops;
    return ETD_OK;
}

int etd_parity_split(const etd_handle* h, int* out) {
    if (!h || !out) return ETD_ERR_CONFIG;
    for (int a = 0; a < h->plan->dim; ++a) out[a] = h->plan->fold[a] ? 1 : 0;
    return ETD_OK;
}

int etd_setup_fold_matrices(int n, int mode, double* ff, double* fb) {
    if (n < 2 || ((n + 1) / 2) % 8 != 0 || (mode != 0 && mode != 1) || !ff || !fb) return ETD_ERR_CONFIG;
    try {
        const etd::AxisOperator op = etd::axis_operator(n, 0.0, 1.0, 1, 1.0, 0.0);
        std::vector<double> Pc, lam, a, b;
        etd::eigensystem(op, Pc, lam);
        etd::fold_matrices(Pc, n, mode, a, b);
        std::memcpy(ff, a.data(), a.size() * 8);
        std::memcpy(fb, b.data(), b.size() * 8);
    } catch (...) {
        return ETD_ERR_CONFIG;
    }
    return ETD_OK;
}

int etd_setup_fold2_matrices(int n, int mode, double* ga, double* gb, double* fb, double* go, double* ge) {
    const int h = (n + 1) / 2;
    if (n < 2 || !(n & 1) || h % 16 != 0 || (mode != 0 && mode != 1) || !ga || !gb || !fb) return ETD_ERR_CONFIG;
    try {
        const etd::AxisOperator op = etd::axis_operator(n, 0.0, 1.0, 1, 1.0, 0.0);
        std::vector<double> Pc, lam, a, b, c, o, e;
        etd::eigensystem(op, Pc, lam);
        etd::fold2_matrices(Pc, n, mode, a, b, c, &o, &e);
        std::memcpy(ga, a.data(), a.size() * 8);
        std::memcpy(gb, b.data(), b.size() * 8);
        std::memcpy(fb, c.data(), c.size() * 8);
        if (go) std::memcpy(go, o.data(), o.size() * 8);
        if (ge) std::memcpy(ge, e.data(), e.size() * 8);
    } catch (...) {
        return ETD_ERR_CONFIG;
    }
    return ETD_OK;
}

int etd_setup_back6_matrix(int n, int mode, double* g6) {
    return guarded(nullptr, [&] {
        const int h = (n + 1) / 2;
        if (n < 3 || !(n & 1) || h % 16 != 0) throw etd::ConfigError("fused level-2 backward needs n = 32m - 1");
        if (mode != 0 && mode != 1) throw etd::ConfigError("mode must be 0 or 1");
        etd::AxisOperator op = etd::axis_operator(n, 0.0, 1.0, 1, 1.0, 0.0);
        std::vector<double> Pc, lam, m6;
        etd::eigensystem(op, Pc, lam);
        etd::back6_matrix(Pc, n, mode, m6);
        std::copy(m6.begin(), m6.end(), g6);
    });
}

int etd_fold_level(const etd_handle* h, int* out) {
    if (!h || !out) return ETD_ERR_CONFIG;
    const auto& p = *h->plan;
    for (int a = 0; a < 3; ++a) out[a] = a < p.dim ? (p.fold2_all && p.fold2[a] ? 2 : p.fold[a] ? 1 : 0) : 0;
    return ETD_OK;
}

// Debugging aid: re-run step op `name` (parity 0 schedule) `reps` times on its
// current inputs and report bitwise differences of output `out` against the
// first re-run (a deterministic kernel reports none).
int etd_debug_repeat_op(etd_handle* h, const char* name, int out, int reps, long long* mismatches, long long* pos,
                        int cap) {
    if (!h || !name || !mismatches) return ETD_ERR_CONFIG;
    return guarded(h, [&] {
        auto& p = *h->plan;
        const etd::Op* op = nullptr;
        for (const auto& o : p.steps[p.cur & 1])
            if ((o.kind == etd::Op::KERNEL || o.kind == etd::Op::SOURCE) && o.name == name) op = &o;
        if (!op || op->kind != etd::Op::KERNEL) throw etd::ConfigError("no such kernel op");
        if (out < 0 || out >= std::max(1, op->L.S)) throw etd::ConfigError("output index beyond the launch's stack");
        // outputs are out_stride apart (pair launches: 2 fields); each is one field
        const long long F = p.slab.F;
        const double* target = op->L.args.out + (size_t)out * op->L.args.out_stride;
        double* ref = nullptr;
        unsigned long long* cnt = nullptr;
        long long* dpos = nullptr;
        ETD_CK(cudaMalloc(&ref, F * 8));
        ETD_CK(cudaMalloc(&cnt, 8));
        ETD_CK(cudaMalloc(&dpos, 8 * std::max(1, cap)));
        etd::run_op(p, *op, p.stream);
        ETD_CK(cudaMemcpyAsync(ref, target, F * 8, cudaMemcpyDeviceToDevice, p.stream));
        *mismatches = 0;
        for (int r = 0; r < reps; ++r) {
            etd::run_op(p, *op, p.stream);
            ETD_CK(cudaMemsetAsync(cnt, 0, 8, p.stream));
            etd::etd_diff_positions<<<1184, 256, 0, p.stream>>>(ref, target, F, cnt, dpos, cap);
            unsigned long long c = 0;
            ETD_CK(cudaMemcpyAsync(&c, cnt, 8, cudaMemcpyDeviceToHost, p.stream));
            ETD_CK(cudaStreamSynchronize(p.stream));
            if ((long long)c > *mismatches) {
                *mismatches = (long long)c;
                if (pos && cap > 0)
                    ETD_CK(cudaMemcpy(pos, dpos, 8 * std::min<long long>(cap, c), cudaMemcpyDeviceToHost));
            }
        }
        cudaFree(ref);
        cudaFree(cnt);
        cudaFree(dpos);
    });
}

int etd_debug_transform(etd_handle* h, int species, int axis, int back, int ell, int apply_q, const double* in,
                        double* out) {
    if (!h || !in || !out) return ETD_ERR_CONFIG;
    return guarded(h, [&] { etd::debug_transform(*h->plan, species, axis, back, ell, apply_q, in, out); });
}

int etd_save_snapshot(etd_handle* h, int species, const char* path) {
    if (!h || !path) return ETD_ERR_CONFIG;
    return guarded(h, [&] { etd::save_snapshot(*h->plan, species, path); });
}

int etd_load_snapshot(etd_handle* h, int species, const char* path, long n) {
    if (!h || !path) return ETD_ERR_CONFIG;
    return guarded(h, [&] { etd::load_snapshot(*h->plan, species, path, n); });
}

int etd_set_source(etd_handle* h, int src_kind, const double* src_params) {
    if (!h) return ETD_ERR_CONFIG;
    return guarded(h, [&] { etd::set_source(*h->plan, src_kind, src_params); });
}

int etd_setup_axis(int n, double low, double high, int dim, double kappa, double q, double* P, double* lambda) {
    if (!P || !lambda) return ETD_ERR_CONFIG;
    return guarded(nullptr, [&] {
        const auto op = etd::axis_operator(n, low, high, dim, kappa, q);
        std::vector<double> pc, lam;
        etd::eigensystem(op, pc, lam);
        std::memcpy(P, pc.data(), pc.size() * 8);
        std::memcpy(lambda, lam.data(), lam.size() * 8);
    });
}

int etd_setup_dvector(int n, const double* lambda, double tau, int family, int ell, double* d) {
    if (!lambda || !d) return ETD_ERR_CONFIG;
    return guarded(nullptr, [&] {
        if (!(tau > 0.0)) throw etd::ConfigError("tau must be positive");
        const auto v = etd::dvector(std::vector<double>(lambda, lambda + n), tau, etd::pade_scheme(family), ell);
        std::memcpy(d, v.data(), v.size() * 8);
    });
}

int etd_setup_scheme(int family, double* out, int* nterms) {
    if (!out || !nterms) return ETD_ERR_CONFIG;
    return guarded(nullptr, [&] {
        const auto s = etd::pade_scheme(family);
        *nterms = (int)s.terms[0].size();
        for (int ell = 0; ell < 3; ++ell)
            for (int t = 0; t < *nterms; ++t) {
                const auto& pr = s.terms[ell][t];
                double* o = out + (ell * (*nterms) + t) * 4;
                o[0] = pr.pole.real(); o[1] = pr.pole.imag(); o[2] = pr.residue.real(); o[3] = pr.residue.imag();
            }
    });
}

int etd_fill_config_ic(int config, unsigned long long seed, int species, int n, int z0, int z1, double* out) {
    if (!out) return ETD_ERR_CONFIG;
    return guarded(nullptr, [&] { etd::fill_config_ic(config, seed, species, n, z0, z1, out); });
}

}  // extern "C"
