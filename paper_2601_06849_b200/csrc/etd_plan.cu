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

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/etd_b200.h"
#include "etd_kernels.cuh"
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
                            const unsigned long long* strides_elems, const unsigned* box) {
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
                             bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    return m;
}

// ------------------------------------------------------------ kernel registry
struct KernelSpec {
    const void* fn;
    int threads, smem, bm, bn, S;
};

template <int MODE, int S, int EPI, bool PRO, int BM, int BN, int WMW, int WNW, int ST>
static KernelSpec make_spec() {
    using Cfg = ContractCfg<MODE, S, EPI, PRO, BM, BN, WMW, WNW, ST>;
    auto k = etd_contract<MODE, S, EPI, PRO, BM, BN, WMW, WNW, ST>;
    return {reinterpret_cast<const void*>(k), Cfg::THREADS, Cfg::SMEM_BYTES, BM, BN, S};
}

template <int MODE, int S, int EPI, bool PRO>
static KernelSpec spec() {
    // Tile shapes: every variant keeps 64 FP64 accumulators per thread (8 warps).
    // Source-prologue kernels use an 8x1 warp grid so that each A element's
    // f(U) is evaluated by exactly one warp (it runs on the shared FP64/DMMA pipe).
    if constexpr (S == 1) return make_spec<MODE, 1, EPI, PRO, 128, 128, 4, 2, 6>();
    else if constexpr (S == 2 && PRO) return make_spec<MODE, 2, EPI, PRO, 64, 128, 8, 1, 8>();
    else if constexpr (S == 2) return make_spec<MODE, 2, EPI, PRO, 64, 128, 2, 4, 6>();
    else if constexpr (PRO) return make_spec<MODE, 4, EPI, PRO, 64, 64, 8, 1, 8>();
    else return make_spec<MODE, 4, EPI, PRO, 64, 64, 2, 4, 5>();
}

static KernelSpec pick(int mode, int S, int epi, bool pro) {
#define ETD_SPEC(M, SS, E, P) \
    if (mode == M && S == SS && epi == E && pro == P) return spec<M, SS, E, P>();
    ETD_SPEC(1, 2, EPI_SCALE, true)
    ETD_SPEC(1, 4, EPI_SCALE, true)
    ETD_SPEC(1, 2, EPI_SCALE, false)
    ETD_SPEC(1, 4, EPI_SCALE, false)
    ETD_SPEC(1, 2, EPI_STORE, false)
    ETD_SPEC(1, 4, EPI_STORE, false)
    ETD_SPEC(1, 1, EPI_SCALE, false)
    ETD_SPEC(1, 1, EPI_STORE, false)
    ETD_SPEC(0, 2, EPI_MIX, false)
    ETD_SPEC(0, 4, EPI_MIX, false)
    ETD_SPEC(0, 1, EPI_WHAT_SRC, false)
    ETD_SPEC(0, 2, EPI_WHAT_SRC, false)
    ETD_SPEC(0, 1, EPI_CORR, false)
    ETD_SPEC(0, 2, EPI_CORR, false)
    ETD_SPEC(0, 1, EPI_UPDATE, false)
    ETD_SPEC(0, 2, EPI_UPDATE, false)
    ETD_SPEC(0, 1, EPI_SCALE, false)
    ETD_SPEC(0, 1, EPI_STORE, false)
#undef ETD_SPEC
    throw ConfigError("no kernel variant for this stage");
}

// ------------------------------------------------------------ the plan
struct Launch {
    std::string name;
    KernelSpec k;
    dim3 grid;
    CUtensorMap tmA, tmB;
    ContractArgs args;
    double flops = 0, bytes = 0;
};

struct StageStat {
    std::string name;
    double ms = 0;
    long launches = 0;
    double flops = 0, bytes = 0;
};

struct Plan {
    etd_desc d{};
    int dim = 2, ns = 1;
    int nx = 1, ny = 1, nz = 1;  // local extents
    int npad[3] = {0, 0, 0};
    long long pitch = 0, plane = 0, F = 0;
    double tau = 0;
    cudaStream_t stream = nullptr;
    double* state[2] = {nullptr, nullptr};
    double* Z = nullptr;
    double* W = nullptr;
    double* PR[3] = {nullptr, nullptr, nullptr};
    double* PTR[3] = {nullptr, nullptr, nullptr};
    double* dvec = nullptr;  // [axis][slot 9][species 2][npadmax]
    int dmax = 0;
    StepStatus* status = nullptr;
    StepStatus* status_host = nullptr;
    int cur = 0;
    std::vector<Launch> steps[2];
    cudaGraphExec_t graph[2] = {nullptr, nullptr};
    bool profiling = false;
    std::vector<StageStat> stats;
    std::string last_msg;
    double last_t = 0;
    long last_step = 0;

    ~Plan() {
        for (auto& g : graph)
            if (g) cudaGraphExecDestroy(g);
        for (auto p : {state[0], state[1], Z, W, dvec}) if (p) cudaFree(p);
        for (int a = 0; a < 3; ++a) {
            if (PR[a]) cudaFree(PR[a]);
            if (PTR[a]) cudaFree(PTR[a]);
        }
        if (status) cudaFree(status);
        if (status_host) cudaFreeHost(status_host);
        if (stream) cudaStreamDestroy(stream);
    }

    const double* dv(int axis, int slot) const {
        return dvec + ((size_t)axis * 9 + slot) * 2 * dmax;
    }
    int n_axis(int a) const { return a == 0 ? nx : a == 1 ? ny : nz; }

    // ---- maps over stacked fields (one TMA box per stage per operand set) ----
    // MODE 0 view: dims {nx, R, count}, box {16, BM, count} -> smem [op][BM][16]
    CUtensorMap mapA_x(const double* base, int count, int bm) const {
        const unsigned long long dims[3] = {(unsigned long long)nx, (unsigned long long)ny * nz,
                                            (unsigned long long)count};
        const unsigned long long st[2] = {(unsigned long long)pitch, (unsigned long long)F};
        const unsigned box[3] = {16, (unsigned)bm, (unsigned)count};
        return make_map(base, 3, dims, st, box);
    }
    // MODE 1 view: dims {x%16, k, x/16, outer, count}, box {16, 16, BM/16, 1, count}
    // -> smem [op][pb][k][16].  x columns past nx read the zero pad of the pitch.
    CUtensorMap mapA_yz(const double* base, int count, bool zaxis, int bm) const {
        const unsigned long long nk = zaxis ? nz : ny, no = zaxis ? ny : nz;
        const unsigned long long sk = zaxis ? plane : pitch, so = zaxis ? pitch : plane;
        const unsigned long long dims[5] = {16, nk, (unsigned long long)((nx + 15) / 16), no,
                                            (unsigned long long)count};
        const unsigned long long st[4] = {sk, 16, so, (unsigned long long)F};
        const unsigned box[5] = {16, 16, (unsigned)(bm / 16), 1, (unsigned)count};
        return make_map(base, 5, dims, st, box);
    }
    // B: row-major n x n (zero-padded to npad).  MODE 0: dims {k, n} box {16, BN};
    // MODE 1: dims {n%16, k, n/16} box {16, 16, BN/16} -> smem [nb][k][16]
    CUtensorMap mapB(const double* M, int axis, int mode, int bn) const {
        const int n = n_axis(axis);
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

    ContractArgs base_args(int axis) const {
        ContractArgs a{};
        a.n_axis = n_axis(axis);
        a.m_extent = axis == 0 ? ny * nz : nx;
        a.zaxis = axis == 2;
        a.nspecies = ns;
        a.pitch = pitch;
        a.plane = plane;
        a.out_stride = F;
        a.aux_stride = F;
        a.dstride = dmax;
        a.src_kind = d.src_kind;
        for (int i = 0; i < 8; ++i) a.sp[i] = d.src_params[i];
        a.ny_local = ny;
        a.gj0 = 0;
        a.gz0 = 0;
        a.status = status;
        a.tau = tau;
        return a;
    }

    // A transform along `axis` of `S` stacked operands at `in` (L loaded), M = P^T (fwd) or P.
    Launch transform(const std::string& name, int axis, bool back, int S, int epi, bool pro,
                     const double* in, double* out) const {
        Launch L;
        L.name = name;
        const int mode = axis == 0 ? 0 : 1;
        L.k = pick(mode, S, epi, pro);
        const int loaded = pro ? S / 2 : S;
        // fwd (M = P^T): mode 0 needs row-major P^T, mode 1 row-major P; back swaps
        const double* M = (mode == 0) != back ? PTR[axis] : PR[axis];
        L.tmA = mode == 0 ? mapA_x(in, loaded, L.k.bm) : mapA_yz(in, loaded, axis == 2, L.k.bm);
        L.tmB = mapB(M, axis, mode, L.k.bn);
        L.args = base_args(axis);
        L.args.out = out;
        const int nax = n_axis(axis);
        const long long mext = L.args.m_extent;
        const unsigned gx = (nax + L.k.bn - 1) / L.k.bn;
        const unsigned gy = (unsigned)((mext + L.k.bm - 1) / L.k.bm);
        const unsigned gz = mode == 0 ? 1u : (axis == 1 ? (unsigned)nz : (unsigned)ny);
        L.grid = dim3(gx, gy, gz);
        const double pts = (double)nx * ny * nz;
        L.flops = 2.0 * nax * pts * S;
        return L;
    }
};

// ------------------------------------------------------------ setup
static int round_up(int x, int m) { return (x + m - 1) / m * m; }

static void check_source(int nspecies, int k) {
    const bool scalar_src = k == ETD_SRC_ZERO || k == ETD_SRC_AC_CUBIC || k == ETD_SRC_POLY3 || k == ETD_SRC_NAN;
    const bool pair_src = k == ETD_SRC_FHN_CUBIC || k == ETD_SRC_FHN_CLASSIC || k == ETD_SRC_MIRROR_AC ||
                          k == ETD_SRC_DECOUPLED || k == ETD_SRC_ZERO;
    if (nspecies == 2 ? !pair_src : !scalar_src)
        throw ConfigError("the CUDA backend needs a device source descriptor matching the plan (no CPU fallback)");
}

static void set_source(Plan& p, int kind, const double* params) {
    check_source(p.ns, kind);
    p.d.src_kind = kind;
    for (int i = 0; i < 8; ++i) p.d.src_params[i] = params ? params[i] : 0.0;
    for (int par = 0; par < 2; ++par) {
        for (auto& L : p.steps[par]) {
            L.args.src_kind = kind;
            for (int i = 0; i < 8; ++i) L.args.sp[i] = p.d.src_params[i];
        }
        if (p.graph[par]) {
            cudaGraphExecDestroy(p.graph[par]);
            p.graph[par] = nullptr;
        }
    }
}

static void build_plan(Plan& p, const etd_desc& d) {
    p.d = d;
    if (d.dim != 2 && d.dim != 3) throw ConfigError("grid dimension must be 2 or 3");
    if (!(d.tau > 0.0)) throw ConfigError("tau must be positive");
    if (d.nspecies != 1 && d.nspecies != 2) throw ConfigError("nspecies must be 1 or 2");
    if (d.family != 0 && d.family != 1) throw ConfigError("unknown Pade family");
    const bool sys = d.nspecies == 2;
    check_source(d.nspecies, d.src_kind);
    if (d.world_size > 1) throw ConfigError("multi-GPU z-slab plans: not available in this build");
    if (sys && !(d.kappa[0] > 0.0 && d.kappa[1] > 0.0))
        throw ConfigError("component diffusivities must be positive");
    p.dim = d.dim;
    p.ns = d.nspecies;
    p.tau = d.tau;
    int dev_count = 0;
    if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0)
        throw NoDevice("no CUDA device visible: the ETD2RK-DS CUDA backend has no CPU fallback");
    ETD_CK(cudaSetDevice(d.device));
    int major = 0;
    ETD_CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d.device));
    if (major != 10) throw NoDevice("this build targets sm_100a (B200)");

    p.nx = d.n[0];
    p.ny = d.n[1];
    p.nz = d.dim == 3 ? d.n[2] : 1;
    for (int a = 0; a < d.dim; ++a)
        if (d.n[a] < 1) throw ConfigError("need at least 2 subintervals for a nonempty interior");
    p.pitch = round_up(p.nx, 32);
    p.plane = p.pitch * p.ny;
    p.F = p.plane * p.nz;
    p.dmax = 0;
    for (int a = 0; a < d.dim; ++a) {
        p.npad[a] = round_up(d.n[a], 32);
        p.dmax = std::max(p.dmax, p.npad[a]);
    }

    ETD_CK(cudaStreamCreateWithFlags(&p.stream, cudaStreamNonBlocking));
    const size_t fb = (size_t)p.F * sizeof(double);
    for (int s = 0; s < 2; ++s) {
        ETD_CK(cudaMalloc(&p.state[s], fb * p.ns));
        ETD_CK(cudaMemsetAsync(p.state[s], 0, fb * p.ns, p.stream));
    }
    ETD_CK(cudaMalloc(&p.Z, fb * 2 * p.ns));
    ETD_CK(cudaMalloc(&p.W, fb * 2 * p.ns));
    ETD_CK(cudaMemsetAsync(p.Z, 0, fb * 2 * p.ns, p.stream));
    ETD_CK(cudaMemsetAsync(p.W, 0, fb * 2 * p.ns, p.stream));

    // per-axis eigensystems and d-vectors (stepper.cpp:118-177; systems use the
    // unit-kappa operator and kappa_c * lambda, system_stepper.cpp:47-61)
    const PadeScheme scheme = pade_scheme(d.family);
    std::vector<double> hd((size_t)3 * 9 * 2 * p.dmax, 0.0);
    for (int a = 0; a < d.dim; ++a) {
        const int n = d.n[a], np = p.npad[a];
        const AxisOperator op = axis_operator(n, d.low[a], d.high[a], d.dim, sys ? 1.0 : d.kappa[0], d.q);
        std::vector<double> Pc, lam;
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
        for (int c = 0; c < p.ns; ++c) {
            std::vector<double> lc(lam);
            if (sys)
                for (auto& x : lc) x *= d.kappa[c];
            const auto d1 = dvector(lc, d.tau, scheme, 1), d2 = dvector(lc, d.tau, scheme, 2),
                       d3 = dvector(lc, d.tau, scheme, 3);
            auto put = [&](int slot, const std::vector<double>& v, double sc) {
                double* o = hd.data() + (((size_t)a * 9 + slot) * 2 + c) * p.dmax;
                for (int i = 0; i < n; ++i) o[i] = sc * v[i];
            };
            // production slots (power-of-two 2 folds exactly; tau folds once)
            put(0, d1, 2.0);
            put(1, d2, 2.0 * d.tau);
            put(2, d3, 2.0 * d.tau);
            // raw and 2x slots for kernel-level tests
            put(3, d1, 1.0); put(4, d2, 1.0); put(5, d3, 1.0);
            put(6, d1, 2.0); put(7, d2, 2.0); put(8, d3, 2.0);
        }
    }
    ETD_CK(cudaMalloc(&p.dvec, hd.size() * 8));
    ETD_CK(cudaMemcpy(p.dvec, hd.data(), hd.size() * 8, cudaMemcpyHostToDevice));
    ETD_CK(cudaMalloc(&p.status, sizeof(StepStatus)));
    ETD_CK(cudaMallocHost(&p.status_host, sizeof(StepStatus)));
    std::memset(p.status_host, 0, sizeof(StepStatus));
    ETD_CK(cudaMemcpy(p.status, p.status_host, sizeof(StepStatus), cudaMemcpyHostToDevice));

    // opt every variant into large dynamic shared memory
    static bool attr_done = false;
    if (!attr_done) {
        for (int mode = 0; mode < 2; ++mode)
            for (int S : {1, 2, 4})
                for (int e = 0; e < 6; ++e)
                    for (int pro = 0; pro < 2; ++pro) {
                        try {
                            KernelSpec ks = pick(mode, S, e, pro != 0);
                            ETD_CK(cudaFuncSetAttribute(ks.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, ks.smem));
                        } catch (const ConfigError&) {
                        }
                    }
        attr_done = true;
    }

    // ---- step schedule per state parity ----
    const int ns = p.ns;
    const long long F = p.F;
    for (int par = 0; par < 2; ++par) {
        auto& L = p.steps[par];
        L.clear();
        const double* in = p.state[par];
        double* out = p.state[1 - par];
        if (p.dim == 3) {
            L.push_back(p.transform("z_fwd_src", 2, false, 2 * ns, EPI_SCALE, true, in, p.Z));
            L.back().args.dA = p.dv(2, 0);
            L.push_back(p.transform("z_back", 2, true, 2 * ns, EPI_STORE, false, p.Z, p.W));
            L.push_back(p.transform("y_fwd", 1, false, 2 * ns, EPI_SCALE, false, p.W, p.Z));
            L.back().args.dA = p.dv(1, 0);
        } else {
            L.push_back(p.transform("y_fwd_src", 1, false, 2 * ns, EPI_SCALE, true, in, p.Z));
            L.back().args.dA = p.dv(1, 0);
        }
        L.push_back(p.transform("y_back", 1, true, 2 * ns, EPI_STORE, false, p.Z, p.W));
        L.push_back(p.transform("x_fwd_mix", 0, false, 2 * ns, EPI_MIX, false, p.W, p.Z));
        L.back().args.dA = p.dv(0, 0);
        L.back().args.dB = p.dv(0, 1);
        L.push_back(p.transform("x_back_src", 0, true, ns, EPI_WHAT_SRC, false, p.Z, p.W));
        L.push_back(p.transform("x_fwd_corr", 0, false, ns, EPI_CORR, false, p.W + ns * F, p.Z));
        L.back().args.aux = p.Z + ns * F;
        L.back().args.dA = p.dv(0, 2);
        L.push_back(p.transform("x_back_upd", 0, true, ns, EPI_UPDATE, false, p.Z, out));
        L.back().args.aux = p.W;
        // algorithmic HBM bytes: operands read + outputs written + aux read
        const double pts = (double)p.nx * p.ny * p.nz * 8.0;
        for (auto& x : L) {
            const int S = x.k.S;
            int loaded = S, outs = S, aux = 0;
            if (x.name.find("_src") != std::string::npos && x.name.rfind("x_", 0) != 0) loaded = S / 2;
            if (x.name == "x_back_src") outs = 2 * S;
            if (x.name == "x_fwd_corr" || x.name == "x_back_upd") aux = S;
            x.bytes = pts * (loaded + outs + aux);
        }
    }
    p.stats.clear();
    for (auto& x : p.steps[0]) p.stats.push_back({x.name, 0, 0, x.flops, x.bytes});
    ETD_CK(cudaStreamSynchronize(p.stream));
}

static void launch(const Plan& p, const Launch& L, cudaStream_t s) {
    void* args[3] = {const_cast<CUtensorMap*>(&L.tmA), const_cast<CUtensorMap*>(&L.tmB),
                     const_cast<ContractArgs*>(&L.args)};
    ETD_CK(cudaLaunchKernel(L.k.fn, L.grid, dim3(L.k.threads), args, L.k.smem, s));
}

static void ensure_graphs(Plan& p) {
    for (int par = 0; par < 2; ++par) {
        if (p.graph[par]) continue;
        cudaGraph_t g;
        ETD_CK(cudaStreamBeginCapture(p.stream, cudaStreamCaptureModeThreadLocal));
        for (auto& L : p.steps[par]) launch(p, L, p.stream);
        ETD_CK(cudaStreamEndCapture(p.stream, &g));
        ETD_CK(cudaGraphInstantiate(&p.graph[par], g, 0));
        cudaGraphDestroy(g);
    }
}

static void copy_status_from_device(Plan& p) {
    ETD_CK(cudaMemcpyAsync(p.status_host, p.status, sizeof(StepStatus), cudaMemcpyDeviceToHost, p.stream));
    ETD_CK(cudaStreamSynchronize(p.stream));
}

static void do_steps(Plan& p, int nsteps) {
    if (nsteps < 0) throw ConfigError("nsteps must be >= 0");
    if (nsteps == 0) return;
    copy_status_from_device(p);
    const long long n_before = p.status_host->n;
    p.status_host->fail = 0;
    p.status_host->cta_done = 0;
    ETD_CK(cudaMemcpyAsync(p.status, p.status_host, sizeof(StepStatus), cudaMemcpyHostToDevice, p.stream));
    if (p.profiling) {
        const size_t nl = p.steps[0].size();
        std::vector<cudaEvent_t> ev((size_t)nsteps * nl + 1);
        for (auto& e : ev) ETD_CK(cudaEventCreate(&e));
        ETD_CK(cudaEventRecord(ev[0], p.stream));
        for (int s = 0; s < nsteps; ++s) {
            const auto& L = p.steps[(p.cur + s) & 1];
            for (size_t i = 0; i < nl; ++i) {
                launch(p, L[i], p.stream);
                ETD_CK(cudaEventRecord(ev[(size_t)s * nl + i + 1], p.stream));
            }
        }
        ETD_CK(cudaStreamSynchronize(p.stream));
        for (int s = 0; s < nsteps; ++s)
            for (size_t i = 0; i < nl; ++i) {
                float ms = 0;
                ETD_CK(cudaEventElapsedTime(&ms, ev[(size_t)s * nl + i], ev[(size_t)s * nl + i + 1]));
                p.stats[i].ms += ms;
                p.stats[i].launches += 1;
            }
        for (auto& e : ev) cudaEventDestroy(e);
    } else {
        ensure_graphs(p);
        for (int s = 0; s < nsteps; ++s) ETD_CK(cudaGraphLaunch(p.graph[(p.cur + s) & 1], p.stream));
    }
    ETD_CK(cudaGetLastError());
    copy_status_from_device(p);
    const long long committed = p.status_host->n - n_before;
    p.cur = (int)((p.cur + committed) & 1);
    if (p.status_host->fail) {
        const int kind = p.status_host->fail;
        const double t = p.status_host->t + (kind >= 2 ? p.tau : 0.0);
        const char* what = kind == 3 ? "step update" : "source";
        throw AbortError(std::string(what) + " produced non-finite values at t=" + std::to_string(t), t,
                         (long)p.status_host->n);
    }
}

static void set_state(Plan& p, int species, const double* host, size_t count, long n, double t) {
    if (species < 0 || species >= p.ns) throw ConfigError("species index out of range");
    if (count != (size_t)p.nx * p.ny * p.nz) throw ConfigError("state shape does not match plan grid");
    double* dst = p.state[p.cur] + (size_t)species * p.F;
    ETD_CK(cudaMemcpy2DAsync(dst, p.pitch * 8, host, (size_t)p.nx * 8, (size_t)p.nx * 8,
                             (size_t)p.ny * p.nz, cudaMemcpyHostToDevice, p.stream));
    p.status_host->n = n;
    p.status_host->t = t;
    p.status_host->fail = 0;
    p.status_host->cta_done = 0;
    ETD_CK(cudaMemcpyAsync(p.status, p.status_host, sizeof(StepStatus), cudaMemcpyHostToDevice, p.stream));
    ETD_CK(cudaStreamSynchronize(p.stream));
}

static void get_state(Plan& p, int species, double* host, size_t count, long* n, double* t) {
    if (species < 0 || species >= p.ns) throw ConfigError("species index out of range");
    if (count != (size_t)p.nx * p.ny * p.nz) throw ConfigError("output shape does not match plan grid");
    const double* src = p.state[p.cur] + (size_t)species * p.F;
    ETD_CK(cudaMemcpy2DAsync(host, (size_t)p.nx * 8, src, p.pitch * 8, (size_t)p.nx * 8,
                             (size_t)p.ny * p.nz, cudaMemcpyDeviceToHost, p.stream));
    copy_status_from_device(p);
    if (n) *n = (long)p.status_host->n;
    if (t) *t = p.status_host->t;
}

static void debug_transform(Plan& p, int species, int axis, int back, int ell, int apply_q,
                            const double* in, double* out) {
    if (axis < 0 || axis >= p.dim) throw ConfigError("axis out of range for field dimension");
    if (species < 0 || species >= p.ns) throw ConfigError("species index out of range");
    if (ell < 0 || ell > 3) throw ConfigError("ell must be 1, 2, or 3");
    const size_t cnt = (size_t)p.nx * p.ny * p.nz;
    ETD_CK(cudaMemcpy2DAsync(p.W, p.pitch * 8, in, (size_t)p.nx * 8, (size_t)p.nx * 8, (size_t)p.ny * p.nz,
                             cudaMemcpyHostToDevice, p.stream));
    p.status_host->fail = 0;
    ETD_CK(cudaMemcpyAsync(p.status, p.status_host, sizeof(StepStatus), cudaMemcpyHostToDevice, p.stream));
    const double* result = nullptr;
    if (apply_q) {
        if (ell < 1) throw ConfigError("apply_q needs ell in 1..3");
        Launch f = p.transform("dbg_fwd", axis, false, 1, EPI_SCALE, false, p.W, p.Z);
        f.args.dA = p.dv(axis, 6 + ell - 1) + species * p.dmax;
        Launch b = p.transform("dbg_back", axis, true, 1, EPI_STORE, false, p.Z, p.W + p.F);
        launch(p, f, p.stream);
        launch(p, b, p.stream);
        result = p.W + p.F;
    } else {
        Launch f = p.transform("dbg", axis, back != 0, 1, ell ? EPI_SCALE : EPI_STORE, false, p.W, p.Z);
        if (ell) f.args.dA = p.dv(axis, 3 + ell - 1) + species * p.dmax;
        launch(p, f, p.stream);
        result = p.Z;
    }
    ETD_CK(cudaGetLastError());
    ETD_CK(cudaMemcpy2DAsync(out, (size_t)p.nx * 8, result, p.pitch * 8, (size_t)p.nx * 8, (size_t)p.ny * p.nz,
                             cudaMemcpyDeviceToHost, p.stream));
    ETD_CK(cudaStreamSynchronize(p.stream));
    (void)cnt;
}

}  // namespace etd

// =================================================================== C-ABI
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
    } catch (const std::bad_alloc& e) {
        if (h) h->msg = "host allocation failed"; else g_create_error = "host allocation failed";
        return ETD_ERR_MEMORY;
    } catch (const std::exception& e) {
        if (h) h->msg = e.what(); else g_create_error = e.what();
        return ETD_ERR_CUDA;
    }
}
}  // namespace

extern "C" {

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

int etd_destroy(etd_handle* h) {
    delete h;
    return ETD_OK;
}

int etd_slab_range(const etd_handle* h, int* z0, int* z1) {
    if (!h) return ETD_ERR_CONFIG;
    if (z0) *z0 = 0;
    if (z1) *z1 = h->plan->nz;
    return ETD_OK;
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
    const size_t cnt = (size_t)p.nx * p.ny * p.nz;
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

int etd_launches_per_step(const etd_handle* h) { return h ? (int)h->plan->steps[0].size() : 0; }

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

int etd_debug_transform(etd_handle* h, int species, int axis, int back, int ell, int apply_q, const double* in,
                        double* out) {
    if (!h || !in || !out) return ETD_ERR_CONFIG;
    return guarded(h, [&] { etd::debug_transform(*h->plan, species, axis, back, ell, apply_q, in, out); });
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
