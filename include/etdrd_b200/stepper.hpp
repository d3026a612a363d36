// etdrd_b200/stepper.hpp — C++ mirror of the reference stepper interface
// (/root/reference/proj/core/include/etdrd/{grid,field,errors,stepper}.hpp) for
// the B200 backend, header-only over the C-ABI in etd_b200.h.
//
// Same names, argument meaning and error behaviour as the reference:
//   Grid / build_grid / unit_box_grid                 grid.hpp:17-47
//   Field (dense FP64, x-fastest)                     field.hpp:13-54
//   ConfigError / NumericsError / StepperAbort / MemoryGuardError   errors.hpp:8-30
//   make_plan / advance / StepperState                stepper.hpp:59-86
//   make_system_plan / etd2rkds_step_system / SystemState  stepper.hpp:91-117
// Differences (documented in INTEGRATION.md): the source is a DeviceSource
// descriptor (a std::function cannot run on the GPU), plans own device memory
// (move-only), make_system_plan accepts 3D grids, and advance_n / step() keep
// the state device-resident across steps.
#pragma once

#include <array>
#include <complex>
#include <cstddef>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../etd_b200.h"

namespace etdrd_b200 {

// ---------------------------------------------------------------- errors.hpp
struct ConfigError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct NumericsError : std::runtime_error { using std::runtime_error::runtime_error; };
struct StepperAbort : std::runtime_error {
    StepperAbort(const std::string& what, double t_abort, long step_abort)
        : std::runtime_error(what), t(t_abort), step(step_abort) {}
    double t = 0.0;
    long step = 0;
};
struct MemoryGuardError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };

namespace detail {
inline void check(int rc, const etd_handle* h) {
    if (rc == ETD_OK) return;
    char msg[1024];
    double t = 0.0;
    long step = 0;
    etd_last_error(h, msg, sizeof msg, &t, &step);
    switch (rc) {
    case ETD_ERR_ABORT: throw StepperAbort(msg, t, step);
    case ETD_ERR_CONFIG: throw ConfigError(msg);
    case ETD_ERR_NUMERICS: throw NumericsError(msg);
    case ETD_ERR_MEMORY: throw MemoryGuardError(msg);
    default: throw DeviceError(msg);
    }
}
}  // namespace detail

// ---------------------------------------------------------------- grid.hpp
enum class Axis : int { X = 0, Y = 1, Z = 2 };

struct Grid {
    int dim = 2;
    std::array<double, 3> low{0.0, 0.0, 0.0};
    std::array<double, 3> high{1.0, 1.0, 1.0};
    std::array<int, 3> m{2, 2, 1};      // SUBINTERVALS per axis; interior = m-1
    std::array<double, 3> h{0.5, 0.5, 1.0};

    int interior(int a) const { return m[a] - 1; }
    std::size_t total_interior() const {
        std::size_t n = 1;
        for (int a = 0; a < dim; ++a) n *= static_cast<std::size_t>(m[a] - 1);
        return n;
    }
    double coord(int a, int i) const { return low[a] + (i + 1) * h[a]; }
    std::array<int, 3> interior_shape() const { return {m[0] - 1, m[1] - 1, dim == 3 ? m[2] - 1 : 1}; }
};

inline Grid build_grid(int dim, std::span<const std::pair<double, double>> bounds, std::span<const int> m_per_axis) {
    if (dim != 2 && dim != 3) throw ConfigError("grid dimension must be 2 or 3, got " + std::to_string(dim));
    if (bounds.size() != static_cast<std::size_t>(dim) || m_per_axis.size() != static_cast<std::size_t>(dim))
        throw ConfigError("bounds/m arrays must have one entry per dimension");
    Grid g;
    g.dim = dim;
    g.m = {1, 1, 1};
    for (int a = 0; a < dim; ++a) {
        auto [lo, hi] = bounds[a];
        if (!(hi > lo)) throw ConfigError("axis " + std::to_string(a) + ": upper bound must exceed lower");
        if (m_per_axis[a] < 2)
            throw ConfigError("axis " + std::to_string(a) + ": need at least 2 subintervals for a nonempty interior");
        g.low[a] = lo;
        g.high[a] = hi;
        g.m[a] = m_per_axis[a];
    }
    for (int a = 0; a < 3; ++a) g.h[a] = (g.high[a] - g.low[a]) / g.m[a];
    return g;
}

inline Grid unit_box_grid(int dim, int m) {
    std::array<std::pair<double, double>, 3> b{{{0.0, 1.0}, {0.0, 1.0}, {0.0, 1.0}}};
    std::array<int, 3> ms{m, m, m};
    return build_grid(dim, std::span(b).first(dim), std::span(ms).first(dim));
}

// ---------------------------------------------------------------- field.hpp
class Field {
public:
    Field() = default;
    Field(int dim, std::array<int, 3> shape)
        : dim_(dim), shape_(shape), data_(static_cast<std::size_t>(shape[0]) * shape[1] * shape[2], 0.0) {}
    static Field zeros(const Grid& g) { return Field(g.dim, g.interior_shape()); }
    int dim() const { return dim_; }
    const std::array<int, 3>& shape() const { return shape_; }
    int nx() const { return shape_[0]; }
    int ny() const { return shape_[1]; }
    int nz() const { return shape_[2]; }
    std::size_t size() const { return data_.size(); }
    double& operator[](std::size_t i) { return data_[i]; }
    double operator[](std::size_t i) const { return data_[i]; }
    double& at(int i, int j, int k = 0) {
        return data_[i + static_cast<std::size_t>(shape_[0]) * (j + static_cast<std::size_t>(shape_[1]) * k)];
    }
    double at(int i, int j, int k = 0) const {
        return data_[i + static_cast<std::size_t>(shape_[0]) * (j + static_cast<std::size_t>(shape_[1]) * k)];
    }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }
    bool same_shape(const Field& o) const { return dim_ == o.dim_ && shape_ == o.shape_; }

private:
    int dim_ = 0;
    std::array<int, 3> shape_{0, 0, 1};
    std::vector<double> data_;
};

// ---------------------------------------------------------------- rational / backend
enum class PadeFamily { P02 = ETD_P02, P04 = ETD_P04 };
enum class BackendKind { Spectral, Thomas, NonSplitBanded, ExactExpReference, CudaSpectral = 100, CudaThomas = 101 };

inline std::string family_name(PadeFamily f) { return f == PadeFamily::P04 ? "p04" : "p02"; }

// rational.hpp:15-47: upper-half-plane pole/residue terms of the three weight
// functions (ell = 1..3), built by the same host setup the device plan uses
// (rational.cpp:133-177; etd_setup_scheme).  A plan made from a RationalScheme
// runs its family (the d-vectors are rebuilt from it on the host).
struct PoleResiduePair {
    std::complex<double> pole;
    std::complex<double> residue;
};
struct RationalScheme {
    PadeFamily name = PadeFamily::P02;
    std::array<std::vector<PoleResiduePair>, 3> terms;  // index ell-1
    const std::vector<PoleResiduePair>& for_ell(int ell) const {
        if (ell < 1 || ell > 3) throw ConfigError("ell must be 1, 2, or 3");
        return terms[ell - 1];
    }
};
inline RationalScheme scheme_by_family(PadeFamily f) {
    double buf[24];
    int nt = 0;
    if (etd_setup_scheme(static_cast<int>(f), buf, &nt) != ETD_OK) throw ConfigError("unknown Pade family");
    RationalScheme s;
    s.name = f;
    for (int ell = 0; ell < 3; ++ell)
        for (int t = 0; t < nt; ++t) {
            const double* e = buf + 4 * (ell * nt + t);
            s.terms[ell].push_back({{e[0], e[1]}, {e[2], e[3]}});
        }
    return s;
}
inline RationalScheme scheme_p02() { return scheme_by_family(PadeFamily::P02); }
inline RationalScheme scheme_p04() { return scheme_by_family(PadeFamily::P04); }

// Device stand-in for SourceFunction / SystemSource (stepper.hpp:18-29).
struct DeviceSource {
    int kind = ETD_SRC_AC_CUBIC;
    std::array<double, 8> params{};
    bool autonomous = true;

    static DeviceSource allen_cahn_cubic() { return {ETD_SRC_AC_CUBIC, {}, true}; }
    static DeviceSource fhn_cubic(double a = 0.1, double eps = 0.01, double beta = 0.5) {
        return {ETD_SRC_FHN_CUBIC, {a, eps, beta}, true};
    }
    static DeviceSource fhn_classic(double eps = 1.0, double alpha = 1.0) {
        return {ETD_SRC_FHN_CLASSIC, {eps, alpha}, true};
    }
    static DeviceSource poly3(double p0, double p1, double p2, double p3) {
        return {ETD_SRC_POLY3, {p0, p1, p2, p3}, true};
    }
    // catalogue Allen-Cahn with manufactured forcing (problems.cpp:68-106)
    static DeviceSource allen_cahn_manufactured(int dim, double lambda = 1.0, double kappa = 1.0) {
        const double pi = 3.14159265358979323846;
        return {ETD_SRC_AC_MANUFACTURED, {lambda, -lambda + kappa * dim * pi * pi, kappa, double(dim)}, false};
    }
    // rho u/(1-u) with the u >= 1 domain guard (problems.cpp:108-136)
    static DeviceSource singular(double rho = 0.1) { return {ETD_SRC_SINGULAR, {rho}, true}; }
};
using SourceFunction = DeviceSource;
using SystemSource = DeviceSource;

// ---------------------------------------------------------------- plans
class PlanHandle {
public:
    PlanHandle() = default;
    explicit PlanHandle(const etd_desc& d) {
        etd_handle* h = nullptr;
        detail::check(etd_create(&d, &h), nullptr);
        h_.reset(h);
    }
    etd_handle* get() const { return h_.get(); }
    explicit operator bool() const { return static_cast<bool>(h_); }

private:
    struct Del { void operator()(etd_handle* h) const { etd_destroy(h); } };
    std::unique_ptr<etd_handle, Del> h_;
};

namespace detail {
inline etd_desc make_desc(const Grid& g, double tau, PadeFamily fam, int ns, double k0, double k1, double q,
                          const DeviceSource& src, int device) {
    etd_desc d{};
    d.dim = g.dim;
    const auto sh = g.interior_shape();
    for (int a = 0; a < 3; ++a) {
        d.n[a] = a < g.dim ? sh[a] : 1;
        d.low[a] = g.low[a];
        d.high[a] = g.high[a];
    }
    d.tau = tau;
    d.family = static_cast<int>(fam);
    d.nspecies = ns;
    d.kappa[0] = k0;
    d.kappa[1] = k1;
    d.q = q;
    d.src_kind = src.kind;
    for (int i = 0; i < 8; ++i) d.src_params[i] = src.params[i];
    d.device = device;
    d.world_size = 1;
    d.rank = 0;
    d.nccl_unique_id = nullptr;
    d.backend = ETD_SPECTRAL;
    return d;
}
// Spectral / CudaSpectral / ExactExpReference -> transforms, Thomas / CudaThomas ->
// tridiagonal solves; NonSplitBanded (banded.cpp) has no device implementation
inline int device_backend(BackendKind b) {
    if (b == BackendKind::Spectral || b == BackendKind::CudaSpectral || b == BackendKind::ExactExpReference)
        return ETD_SPECTRAL;
    if (b == BackendKind::Thomas || b == BackendKind::CudaThomas) return ETD_THOMAS;
    throw ConfigError("etdrd_b200 implements the Spectral, Thomas and ExactExpReference backends");
}
inline void set_source(etd_handle* h, const DeviceSource& s) {
    check(etd_set_source(h, s.kind, s.params.data()), h);
}
}  // namespace detail

struct StepperPlan {
    Grid grid;
    double tau = 0.0, kappa = 1.0, q = 0.0;
    PadeFamily scheme = PadeFamily::P02;
    BackendKind backend = BackendKind::CudaSpectral;
    PlanHandle handle;
};

struct StepperState {
    long n = 0;
    double t = 0.0;
    Field U;
};

// stepper.hpp:59-61.  Spectral, Thomas and ExactExpReference backends on the device.
// memory_cap_bytes caps the plan's device memory on this GPU (0 = the free memory);
// a plan above it throws MemoryGuardError before allocating (the reference guards
// its banded factorisation the same way, stepper.cpp:57-70).
inline StepperPlan make_plan(const Grid& grid, double tau, double kappa, double q, PadeFamily scheme,
                             BackendKind backend = BackendKind::CudaSpectral, std::size_t memory_cap_bytes = 0,
                             int device = 0) {
    const int bk = detail::device_backend(backend);
    StepperPlan p;
    p.backend = backend;
    p.grid = grid;
    p.tau = tau;
    p.kappa = kappa;
    p.q = q;
    p.scheme = scheme;
    etd_desc d = detail::make_desc(grid, tau, scheme, 1, kappa, 0.0, q, DeviceSource::allen_cahn_cubic(), device);
    d.backend = bk;
    // BackendKind::ExactExpReference (stepper.cpp:145-170, 259-295): the same step
    // with exact e^{-tau lambda}, phi1, phi2 multipliers
    if (backend == BackendKind::ExactExpReference) d.family = ETD_EXACT;
    d.memory_cap_bytes = memory_cap_bytes;
    p.handle = PlanHandle(d);
    return p;
}
// The reference signature (stepper.hpp:59-61): scheme as a RationalScheme value.
inline StepperPlan make_plan(const Grid& grid, double tau, double kappa, double q, const RationalScheme& scheme,
                             BackendKind backend, std::size_t memory_cap_bytes = 0) {
    return make_plan(grid, tau, kappa, q, scheme.name, backend, memory_cap_bytes);
}

// stepper.hpp:85-86 value semantics; nsteps > 1 keeps the state on the device
// between steps (StepperAbort reports the failing step's input t and n).
inline StepperState advance(const StepperPlan& plan, const StepperState& state, const SourceFunction& f,
                            int nsteps = 1) {
    etd_handle* h = plan.handle.get();
    if (state.U.shape() != plan.grid.interior_shape()) throw ConfigError("state shape does not match plan grid");
    detail::set_source(h, f);
    StepperState out{0, 0.0, Field(state.U.dim(), state.U.shape())};
    detail::check(etd_advance(h, state.U.data(), nullptr, state.n, state.t, nsteps, out.U.data(), nullptr, &out.n,
                              &out.t),
                  h);
    return out;
}

// stepper.cpp:182-257: the split steps `advance` dispatches to (one step each).
inline StepperState etd2rkds_step_2d(const StepperPlan& plan, const StepperState& state, const SourceFunction& f) {
    if (plan.grid.dim != 2) throw ConfigError("2D step on non-2D plan");
    if (plan.backend == BackendKind::ExactExpReference)
        throw ConfigError("2D split step requires the spectral or thomas backend");
    return advance(plan, state, f);
}
inline StepperState etd2rkds_step_3d(const StepperPlan& plan, const StepperState& state, const SourceFunction& f) {
    if (plan.grid.dim != 3) throw ConfigError("3D step on non-3D plan");
    if (plan.backend == BackendKind::ExactExpReference)
        throw ConfigError("3D split step requires the spectral or thomas backend");
    return advance(plan, state, f);
}
// stepper.hpp:76-77 / stepper.cpp:259-295: the exact-exponential step, on plans made
// with BackendKind::ExactExpReference (no 64-points-per-axis cap on the device).
inline StepperState etd2rkds_reference_step(const StepperPlan& plan, const StepperState& state,
                                            const SourceFunction& f) {
    if (plan.backend != BackendKind::ExactExpReference) throw ConfigError("reference step requires the exact backend");
    return advance(plan, state, f);
}

// stepper.cpp:38-46
inline double phi1(double x) { return etd_setup_phi(1, x); }
inline double phi2(double x) { return etd_setup_phi(2, x); }

struct SystemPlan {
    Grid grid;
    double tau = 0.0, kappa_u = 1.0, kappa_v = 1.0, q = 0.0;
    PadeFamily scheme = PadeFamily::P02;
    BackendKind backend = BackendKind::CudaSpectral;
    PlanHandle handle;
};

struct SystemState {
    long n = 0;
    double t = 0.0;
    Field U, V;
};

// stepper.hpp:107-108; 2D and 3D (the reference throws for dim != 2).
inline SystemPlan make_system_plan(const Grid& grid, double tau, double kappa_u, double kappa_v, double q,
                                   PadeFamily scheme, BackendKind backend = BackendKind::CudaSpectral,
                                   int device = 0) {
    if (backend == BackendKind::ExactExpReference)
        throw ConfigError("system plans support the spectral and thomas backends only");
    const int bk = detail::device_backend(backend);
    SystemPlan p;
    p.backend = backend;
    p.grid = grid;
    p.tau = tau;
    p.kappa_u = kappa_u;
    p.kappa_v = kappa_v;
    p.q = q;
    p.scheme = scheme;
    etd_desc d = detail::make_desc(grid, tau, scheme, 2, kappa_u, kappa_v, q, DeviceSource::fhn_cubic(), device);
    d.backend = bk;
    p.handle = PlanHandle(d);
    return p;
}

// The reference signature (stepper.hpp:107-108): scheme as a RationalScheme value.
inline SystemPlan make_system_plan(const Grid& grid, double tau, double kappa_u, double kappa_v, double q,
                                   const RationalScheme& scheme, BackendKind backend) {
    if (backend == BackendKind::ExactExpReference || backend == BackendKind::NonSplitBanded)
        throw ConfigError("system plans support the spectral and thomas backends only");
    return make_system_plan(grid, tau, kappa_u, kappa_v, q, scheme.name, backend);
}

// system_stepper.cpp:74-114
inline SystemState etd2rkds_step_system(const SystemPlan& plan, const SystemState& state, const SystemSource& f,
                                        int nsteps = 1) {
    etd_handle* h = plan.handle.get();
    if (state.U.shape() != plan.grid.interior_shape() || !state.U.same_shape(state.V))
        throw ConfigError("system state shape does not match plan grid");
    detail::set_source(h, f);
    SystemState out{0, 0.0, Field(state.U.dim(), state.U.shape()), Field(state.V.dim(), state.V.shape())};
    detail::check(etd_advance(h, state.U.data(), state.V.data(), state.n, state.t, nsteps, out.U.data(),
                              out.V.data(), &out.n, &out.t),
                  h);
    return out;
}

}  // namespace etdrd_b200
