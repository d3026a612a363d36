// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A thin extern "C" driver over the UNMODIFIED reference library (etdrd,
// /root/reference/proj/core/src/*.cpp, compiled out-of-tree by oracle/Makefile
// into oracle/_ref/libetdrd_ref.so).  It lets the Python test-suite and the
// bench's CPU arm run the reference's own stepping code on host arrays:
//   * scalar 2D/3D: make_plan (stepper.cpp:118-177) + advance (stepper.cpp:318-331)
//   * two-species 2D: make_system_plan + etd2rkds_step_system (system_stepper.cpp:31-114)
//   * two-species 3D: the reference has no 3D system stepper (system_stepper.cpp:33
//     throws for dim != 2), so the step is composed from reference public
//     primitives exactly as system_stepper.cpp:80-111 with the 3D z->y filter of
//     stepper.cpp:244-247.
// Source terms are pointwise functors plugged into the reference SourceFunction /
// SystemSource interfaces (stepper.hpp:18-29), as its own tests do
// (proj/tests/test_stepper.cpp:451-472).
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <string>

#include "etdrd/errors.hpp"
#include "etdrd/grid.hpp"
#include "etdrd/operators.hpp"
#include "etdrd/problems.hpp"
#include "etdrd/rational.hpp"
#include "etdrd/stepper.hpp"
#include "etdrd/tensor_ops.hpp"
#ifdef REF_HAS_HARNESS
#include "etdrd/harness.hpp"
#endif

using namespace etdrd;

extern "C" {
void scipy_openblas_set_num_threads64_(int);
int scipy_openblas_get_num_threads64_(void);
char* scipy_openblas_get_config64_(void);
}

namespace {

// source kinds shared with paper_2601_06849_b200 (include/etd_b200.h ETD_SRC_*)
enum {
    SRC_ZERO = 0, SRC_AC_CUBIC = 1, SRC_POLY3 = 2, SRC_NAN = 3, SRC_AC_MANUFACTURED = 4, SRC_SINGULAR = 5,
    SRC_FHN_CUBIC = 10, SRC_FHN_CLASSIC = 11, SRC_MIRROR_AC = 12, SRC_DECOUPLED = 13
};

double scalar_f(int kind, const double* p, double u) {
    switch (kind) {
    case SRC_ZERO: return 0.0;
    case SRC_AC_CUBIC: return u - u * u * u;
    case SRC_POLY3: return ((p[3] * u + p[2]) * u + p[1]) * u + p[0];
    default: return 0.0;
    }
}

SourceFunction make_scalar_source(int kind, const double* params, int dim = 2) {
    double p[8] = {0};
    if (params) std::memcpy(p, params, sizeof p);
    // catalogue sources: the reference's own functors (problems.cpp:68-136)
    if (kind == SRC_AC_MANUFACTURED) {
        ProblemParams pp;
        pp.lambda = p[0];
        pp.kappa = p[2];
        return allen_cahn(dim, pp).source;
    }
    if (kind == SRC_SINGULAR) {
        ProblemParams pp;
        pp.rho = p[0];
        return singular_source(dim, pp).source;
    }
    return {[kind, p](double, const Field& u, const Grid&) {
                Field f(u.dim(), u.shape());
                for (std::size_t i = 0; i < f.size(); ++i) f[i] = scalar_f(kind, p, u[i]);
                if (kind == SRC_NAN && f.size() > 0) f[0] = std::numeric_limits<double>::quiet_NaN();
                return f;
            },
            true};
}

SystemSource make_system_source(int kind, const double* params) {
    double p[8] = {0};
    if (params) std::memcpy(p, params, sizeof p);
    return {[kind, p](double t, const Field& U, const Field& V, const Grid&) {
        Field fu(U.dim(), U.shape()), fv(V.dim(), V.shape());
        for (std::size_t i = 0; i < U.size(); ++i) {
            const double u = U[i], v = V[i];
            switch (kind) {
            case SRC_FHN_CUBIC:  // u(1-u)(u-a) - v ; eps*(beta*u - v)
                fu[i] = u * (1.0 - u) * (u - p[0]) - v;
                fv[i] = p[1] * (p[2] * u - v);
                break;
            case SRC_FHN_CLASSIC:  // problems.cpp:170-171
                fu[i] = u - u * u * u / 3.0 - v;
                fv[i] = p[0] * (u - p[1] * v);
                break;
            case SRC_MIRROR_AC:  // test_stepper.cpp:432-438
                fu[i] = u - u * u * u;
                fv[i] = v - v * v * v;
                break;
            case SRC_DECOUPLED:  // u - u^3 ; p0*v + p1 (autonomous variant of test_stepper.cpp:451-456)
                fu[i] = u - u * u * u;
                fv[i] = p[0] * v + p[1];
                break;
            default:
                fu[i] = 0.0;
                fv[i] = 0.0;
            }
        }
        (void)t;
        return std::make_pair(std::move(fu), std::move(fv));
    }};
}

void put_err(char* err, int errlen, const std::string& s) {
    if (err && errlen > 0) {
        std::strncpy(err, s.c_str(), errlen - 1);
        err[errlen - 1] = 0;
    }
}

Field field_from(const Grid& g, const double* src) {
    Field f = Field::zeros(g);
    std::memcpy(f.data(), src, f.size() * sizeof(double));
    return f;
}

// 3D (or 2D) two-species plan composed from reference primitives
// (system_stepper.cpp:47-61 generalised to dim 3).
struct SysPlan3 {
    Grid grid;
    double tau;
    std::array<std::shared_ptr<const SpectralFactor>, 3> fac;
    std::array<SpectralAxisPayload, 3> pu, pv;
    bool thomas = false;  // BackendKind::Thomas payloads (system_stepper.cpp:62-64)
    std::array<ThomasAxisPayload, 3> tu, tv;

    Field Q(int c, int ell, const Field& g, Axis ax) const {
        const int a = axis_index(ax);
        if (thomas) return apply_Q_thomas(c == 0 ? tu[a] : tv[a], ell, tau, g, ax);
        return apply_Q_spectral(c == 0 ? pu[a] : pv[a], ell, tau, g, ax);
    }
};

SysPlan3 make_sys3(const Grid& g, double tau, double ku, double kv, double q,
                   const RationalScheme& scheme, BackendKind backend = BackendKind::Spectral) {
    SysPlan3 sp;
    sp.grid = g;
    sp.tau = tau;
    sp.thomas = backend == BackendKind::Thomas;
    for (int a = 0; a < g.dim; ++a) {
        auto op = build_operator(g, static_cast<Axis>(a), 1.0, q);
        if (sp.thomas) {
            sp.tu[a] = build_thomas_payload(op, tau, scheme, ku);
            sp.tv[a] = build_thomas_payload(op, tau, scheme, kv);
            continue;
        }
        sp.fac[a] = std::make_shared<const SpectralFactor>(spectral_factor(op));
        const auto& lam = sp.fac[a]->eigvals;
        std::vector<double> lu(lam.size()), lv(lam.size());
        for (std::size_t k = 0; k < lam.size(); ++k) {
            lu[k] = ku * lam[k];
            lv[k] = kv * lam[k];
        }
        sp.pu[a] = build_spectral_payload(sp.fac[a], tau, scheme, lu);
        sp.pv[a] = build_spectral_payload(sp.fac[a], tau, scheme, lv);
    }
    return sp;
}

// system_stepper.cpp:74-114 with the 3D z->y stage-input filter of stepper.cpp:244-247
SystemState sys3_step(const SysPlan3& sp, const SystemState& st, const SystemSource& f) {
    const double t = st.t, tau = sp.tau;
    auto Q = [&](int c, int ell, const Field& g, Axis ax) { return sp.Q(c, ell, g, ax); };
    auto chk = [&](const Field& a, const Field& b, const char* what, double tt) {
        if (!a.all_finite() || !b.all_finite())
            throw StepperAbort(std::string(what) + " produced non-finite values", tt, st.n);
    };
    auto [fu, fv] = f.fn(t, st.U, st.V, sp.grid);
    chk(fu, fv, "source", t);
    auto filt = [&](int c, const Field& g) { return Q(c, 1, Q(c, 1, g, Axis::Z), Axis::Y); };
    const Field w1u = filt(0, st.U), w2u = filt(0, fu);
    const Field w1v = filt(1, st.V), w2v = filt(1, fv);
    auto predict = [&](int c, const Field& w1, const Field& w2) {
        Field W = Q(c, 1, w1, Axis::X);
        const Field lin = Q(c, 2, w2, Axis::X);
        for (std::size_t i = 0; i < W.size(); ++i) W[i] += tau * lin[i];
        return W;
    };
    const Field Wu = predict(0, w1u, w2u), Wv = predict(1, w1v, w2v);
    auto [gu, gv] = f.fn(t + tau, Wu, Wv, sp.grid);
    chk(gu, gv, "source", t + tau);
    for (std::size_t i = 0; i < gu.size(); ++i) gu[i] -= w2u[i];
    for (std::size_t i = 0; i < gv.size(); ++i) gv[i] -= w2v[i];
    Field U1 = Wu, V1 = Wv;
    {
        const Field cu = Q(0, 3, gu, Axis::X);
        for (std::size_t i = 0; i < U1.size(); ++i) U1[i] += tau * cu[i];
        const Field cv = Q(1, 3, gv, Axis::X);
        for (std::size_t i = 0; i < V1.size(); ++i) V1[i] += tau * cv[i];
    }
    chk(U1, V1, "step update", t + tau);
    return {st.n + 1, (st.n + 1) * tau, std::move(U1), std::move(V1)};
}

// Same step as sys3_step (identical reference calls and arithmetic order), with
// explicit lifetimes so that a 1023^3 two-species step fits in ~10 fields of
// host RAM instead of ~18: intermediates are released as soon as the
// reference step would no longer read them.
SystemState sys3_step_lean(const SysPlan3& sp, SystemState st, const SystemSource& f) {
    const double t = st.t, tau = sp.tau;
    auto Q = [&](int c, int ell, const Field& g, Axis ax) { return sp.Q(c, ell, g, ax); };
    auto chk = [&](const Field& a, const Field& b, const char* what, double tt) {
        if (!a.all_finite() || !b.all_finite())
            throw StepperAbort(std::string(what) + " produced non-finite values", tt, st.n);
    };
    Field Wc[2], w2[2];
    {
        auto [fu, fv] = f.fn(t, st.U, st.V, sp.grid);
        chk(fu, fv, "source", t);
        Field* F[2] = {&fu, &fv};
        const Field* X[2] = {&st.U, &st.V};
        for (int c = 0; c < 2; ++c) {
            Field w1 = Q(c, 1, Q(c, 1, *X[c], Axis::Z), Axis::Y);
            w2[c] = Q(c, 1, Q(c, 1, *F[c], Axis::Z), Axis::Y);
            *F[c] = Field();  // f(U) no longer needed
            Wc[c] = Q(c, 1, w1, Axis::X);
            w1 = Field();
            const Field lin = Q(c, 2, w2[c], Axis::X);
            for (std::size_t i = 0; i < Wc[c].size(); ++i) Wc[c][i] += tau * lin[i];
        }
    }
    st.U = Field();
    st.V = Field();
    auto [gu, gv] = f.fn(t + tau, Wc[0], Wc[1], sp.grid);
    chk(gu, gv, "source", t + tau);
    Field* G[2] = {&gu, &gv};
    for (int c = 0; c < 2; ++c) {
        for (std::size_t i = 0; i < G[c]->size(); ++i) (*G[c])[i] -= w2[c][i];
        w2[c] = Field();
        const Field corr = Q(c, 3, *G[c], Axis::X);
        *G[c] = Field();
        for (std::size_t i = 0; i < Wc[c].size(); ++i) Wc[c][i] += tau * corr[i];
    }
    chk(Wc[0], Wc[1], "step update", t + tau);
    return {st.n + 1, (st.n + 1) * tau, std::move(Wc[0]), std::move(Wc[1])};
}

int map_exc(const std::exception& e, char* err, int errlen, double* t_abort, long* step_abort) {
    put_err(err, errlen, e.what());
    if (auto* sa = dynamic_cast<const StepperAbort*>(&e)) {
        if (t_abort) *t_abort = sa->t;
        if (step_abort) *step_abort = sa->step;
        return 3;
    }
    if (dynamic_cast<const ConfigError*>(&e)) return 1;
    if (dynamic_cast<const NumericsError*>(&e)) return 2;
    if (dynamic_cast<const MemoryGuardError*>(&e)) return 4;
    return 5;
}

}  // namespace

extern "C" {

void ref_set_threads(int n) { scipy_openblas_set_num_threads64_(n); }
int ref_get_threads(void) { return scipy_openblas_get_num_threads64_(); }
const char* ref_blas_config(void) { return scipy_openblas_get_config64_(); }

// Scalar run: unit_box_grid(dim, n+1) (grid.hpp:14-16: m counts subintervals),
// make_plan + `nsteps` x advance.  u is x-fastest n^dim, updated in place.
int ref_scalar_run(int dim, int n, double tau, double kappa, double q, int family,
                   int backend, int src_kind, const double* src_params, double* u, long* n_io,
                   double* t_io, int nsteps, double* seconds, char* err, int errlen,
                   double* t_abort, long* step_abort) {
    try {
        const Grid g = unit_box_grid(dim, n + 1);
        const auto plan = make_plan(g, tau, kappa, q,
                                    scheme_by_family(family ? PadeFamily::P04 : PadeFamily::P02),
                                    static_cast<BackendKind>(backend));
        const auto src = make_scalar_source(src_kind, src_params, dim);
        StepperState st{*n_io, *t_io, field_from(g, u)};
        const auto t0 = std::chrono::steady_clock::now();
        for (int s = 0; s < nsteps; ++s) st = advance(plan, st, src);
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        std::memcpy(u, st.U.data(), st.U.size() * sizeof(double));
        *n_io = st.n;
        *t_io = st.t;
        return 0;
    } catch (const std::exception& e) {
        return map_exc(e, err, errlen, t_abort, step_abort);
    }
}

// Two-species run.  dim==2 uses the reference make_system_plan/etd2rkds_step_system
// unchanged; dim==3 uses the composition above (use_composed=1 forces it in 2D too).
int ref_system_run(int dim, int n, double tau, double ku, double kv, double q, int family,
                   int backend, int src_kind, const double* src_params, double* u, double* v, long* n_io,
                   double* t_io, int nsteps, int use_composed, double* seconds, char* err,
                   int errlen, double* t_abort, long* step_abort) {
    try {
        const Grid g = unit_box_grid(dim, n + 1);
        const auto scheme = scheme_by_family(family ? PadeFamily::P04 : PadeFamily::P02);
        const auto src = make_system_source(src_kind, src_params);
        SystemState st{*n_io, *t_io, field_from(g, u), field_from(g, v)};
        std::chrono::steady_clock::time_point t0, t1;
        const auto bk = static_cast<BackendKind>(backend);
        if (dim == 2 && !use_composed) {
            const auto plan = make_system_plan(g, tau, ku, kv, q, scheme, bk);
            t0 = std::chrono::steady_clock::now();
            for (int s = 0; s < nsteps; ++s) st = etd2rkds_step_system(plan, st, src);
            t1 = std::chrono::steady_clock::now();
        } else {
            if (dim == 2) {
                // 2D composed variant: identical to etd2rkds_step_system without the z filter
                const auto plan = make_system_plan(g, tau, ku, kv, q, scheme, bk);
                t0 = std::chrono::steady_clock::now();
                for (int s = 0; s < nsteps; ++s) st = etd2rkds_step_system(plan, st, src);
                t1 = std::chrono::steady_clock::now();
            } else {
                const auto sp = make_sys3(g, tau, ku, kv, q, scheme, bk);
                t0 = std::chrono::steady_clock::now();
                if (use_composed == 2)
                    for (int s = 0; s < nsteps; ++s) st = sys3_step_lean(sp, std::move(st), src);
                else
                    for (int s = 0; s < nsteps; ++s) st = sys3_step(sp, st, src);
                t1 = std::chrono::steady_clock::now();
            }
        }
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        std::memcpy(u, st.U.data(), st.U.size() * sizeof(double));
        std::memcpy(v, st.V.data(), st.V.size() * sizeof(double));
        *n_io = st.n;
        *t_io = st.t;
        return 0;
    } catch (const std::exception& e) {
        return map_exc(e, err, errlen, t_abort, step_abort);
    }
}

// Bounded CPU sample of ONE reference step at full pencil length n (bench.py
// cpu_baseline / --impl reference).  A full-size 3D step at n=1023 needs
// ~140 GiB and minutes on the box's host, so the reference step is run on a
// z-sub-box (n, n, nsub) — its x and y applies are exactly the full-grid
// per-point work — and its z-direction applies (2 per species: Qz1 of U and of
// f(U), stepper.cpp:244-247) are re-timed on an (n, nsub, n) block whose z
// pencils have the full length n.  Estimated per-step time on the sample's
// points:  t_step(sub) - nz_applies*t_z(sub) + nz_applies*t_z(full-length).
// Scalar plans (nspecies=1) use make_plan+advance, systems the composed step.
int ref_sample_step(int n, int nsub, int nspecies, double tau, double k0, double k1, double q, int family,
                    int src_kind, const double* src_params, double* out_seconds, double* out_points,
                    double* parts /* [t_sub, t_zsub, t_zfull] */, char* err, int errlen) {
    try {
        const auto scheme = scheme_by_family(family ? PadeFamily::P04 : PadeFamily::P02);
        const std::array<std::pair<double, double>, 3> b{{{0.0, 1.0}, {0.0, 1.0}, {0.0, 1.0}}};
        const std::array<int, 3> msub{n + 1, n + 1, nsub + 1}, mz{n + 1, nsub + 1, n + 1};
        const Grid gs = build_grid(3, b, msub), gz = build_grid(3, b, mz);
        auto fill = [](const Grid& g, unsigned seed) {
            Field f = Field::zeros(g);
            unsigned long long x = seed * 0x9E3779B97F4A7C15ull + 1;
            for (std::size_t i = 0; i < f.size(); ++i) {
                x ^= x << 13; x ^= x >> 7; x ^= x << 17;
                f[i] = 0.5 * static_cast<double>(x >> 11) * 0x1.0p-53;
            }
            return f;
        };
        using clk = std::chrono::steady_clock;
        auto secs = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); };
        double t_sub, t_zs, t_zf;
        int z_applies;
        if (nspecies == 1) {
            const auto plan = make_plan(gs, tau, k0, q, scheme, BackendKind::Spectral);
            const auto src = make_scalar_source(src_kind, src_params);
            StepperState st{0, 0.0, fill(gs, 1)};
            auto t0 = clk::now();
            st = advance(plan, st, src);
            t_sub = secs(t0, clk::now());
            const auto& pz = plan.spectral[2];
            const Field a = fill(gs, 2);
            t0 = clk::now();
            (void)apply_Q_spectral(pz, 1, tau, a, Axis::Z);
            t_zs = secs(t0, clk::now());
            const auto planz = make_plan(gz, tau, k0, q, scheme, BackendKind::Spectral);
            const Field c = fill(gz, 3);
            t0 = clk::now();
            (void)apply_Q_spectral(planz.spectral[2], 1, tau, c, Axis::Z);
            t_zf = secs(t0, clk::now());
            z_applies = 2;
        } else {
            const auto sp = make_sys3(gs, tau, k0, k1, q, scheme);
            const auto src = make_system_source(src_kind, src_params);
            SystemState st{0, 0.0, fill(gs, 1), fill(gs, 4)};
            auto t0 = clk::now();
            st = sys3_step(sp, st, src);
            t_sub = secs(t0, clk::now());
            const Field a = fill(gs, 2);
            t0 = clk::now();
            (void)apply_Q_spectral(sp.pu[2], 1, tau, a, Axis::Z);
            t_zs = secs(t0, clk::now());
            const auto spz = make_sys3(gz, tau, k0, k1, q, scheme);
            const Field c = fill(gz, 3);
            t0 = clk::now();
            (void)apply_Q_spectral(spz.pu[2], 1, tau, c, Axis::Z);
            t_zf = secs(t0, clk::now());
            z_applies = 4;
        }
        *out_seconds = t_sub - z_applies * t_zs + z_applies * t_zf;
        *out_points = static_cast<double>(n) * n * nsub * nspecies;
        if (parts) { parts[0] = t_sub; parts[1] = t_zs; parts[2] = t_zf; }
        return 0;
    } catch (const std::exception& e) {
        return map_exc(e, err, errlen, nullptr, nullptr);
    }
}

// field.cpp:46-81 (format cross-check of device snapshots)
int ref_save_field(int dim, int nx, int ny, int nz, const double* data, double t, const char* path, char* err,
                   int errlen) {
    try {
        Field f(dim, {nx, ny, nz});
        std::memcpy(f.data(), data, f.size() * sizeof(double));
        save_field(f, t, path);
        return 0;
    } catch (const std::exception& e) {
        return map_exc(e, err, errlen, nullptr, nullptr);
    }
}

int ref_load_field(const char* path, double* data, long long cap, int* shape, double* t, char* err, int errlen) {
    try {
        auto [f, tt] = load_field(path);
        if ((long long)f.size() > cap) throw ConfigError("buffer too small");
        std::memcpy(data, f.data(), f.size() * sizeof(double));
        shape[0] = f.dim(); shape[1] = f.nx(); shape[2] = f.ny(); shape[3] = f.nz();
        *t = tt;
        return 0;
    } catch (const std::exception& e) {
        return map_exc(e, err, errlen, nullptr, nullptr);
    }
}

// operators.cpp:11-34 on unit_box_grid(dim, n+1)
int ref_operator(int dim, int n, int axis, double kappa, double q, double* diag, double* off,
                 char* err, int errlen) {
    try {
        const auto op = build_operator(unit_box_grid(dim, n + 1), static_cast<Axis>(axis), kappa, q);
        *diag = op.diag;
        *off = op.off;
        return 0;
    } catch (const std::exception& e) {
        return map_exc(e, err, errlen, nullptr, nullptr);
    }
}

// operators.cpp:36-56: P column-major n*n, ascending eigenvalues
int ref_spectral_factor(int n, double diag, double off, double* P, double* eig) {
    ToeplitzTridiagOperator op;
    op.n = n;
    op.diag = diag;
    op.off = off;
    const auto f = spectral_factor(op);
    std::memcpy(P, f.P.data(), f.P.size() * sizeof(double));
    std::memcpy(eig, f.eigvals.data(), f.eigvals.size() * sizeof(double));
    return 0;
}

// rational.cpp:187-198
int ref_dvector(int n, const double* eig, double tau, int family, int ell, double* d) {
    const auto scheme = scheme_by_family(family ? PadeFamily::P04 : PadeFamily::P02);
    const auto v = dvector_values(std::span<const double>(eig, n), tau, scheme, ell);
    std::memcpy(d, v.data(), v.size() * sizeof(double));
    return 0;
}

// rational.cpp:133-177: out[ell-1][term] = {pole.re, pole.im, res.re, res.im}
int ref_scheme(int family, double* out, int* nterms) {
    const auto s = scheme_by_family(family ? PadeFamily::P04 : PadeFamily::P02);
    *nterms = static_cast<int>(s.terms[0].size());
    for (int ell = 0; ell < 3; ++ell)
        for (int k = 0; k < *nterms; ++k) {
            const auto& t = s.terms[ell][k];
            double* o = out + (ell * (*nterms) + k) * 4;
            o[0] = t.pole.real();
            o[1] = t.pole.imag();
            o[2] = t.residue.real();
            o[3] = t.residue.imag();
        }
    return 0;
}

// tensor_ops.cpp:107-119 on an (nx,ny,nz) field; M column-major n*n
int ref_contract_axis(int dim, int nx, int ny, int nz, const double* M, int n, const double* in,
                      int axis, int transpose, double* out, char* err, int errlen) {
    try {
        Field f(dim, {nx, ny, nz});
        std::memcpy(f.data(), in, f.size() * sizeof(double));
        const auto r = contract_axis(std::span<const double>(M, static_cast<std::size_t>(n) * n),
                                     n, f, static_cast<Axis>(axis), transpose != 0);
        std::memcpy(out, r.data(), r.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return map_exc(e, err, errlen, nullptr, nullptr);
    }
}

// tensor_ops.cpp:164-172 via a fresh payload (tensor_ops.cpp:144-162)
int ref_apply_q(int dim, int n, double tau, double kappa, double q, int family, int ell,
                int axis, const double* in, double* out, char* err, int errlen) {
    try {
        const Grid g = unit_box_grid(dim, n + 1);
        const auto op = build_operator(g, static_cast<Axis>(axis), kappa, q);
        auto fac = std::make_shared<const SpectralFactor>(spectral_factor(op));
        const auto pay = build_spectral_payload(
            fac, tau, scheme_by_family(family ? PadeFamily::P04 : PadeFamily::P02));
        const Field r = apply_Q_spectral(pay, ell, tau, field_from(g, in), static_cast<Axis>(axis));
        std::memcpy(out, r.data(), r.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return map_exc(e, err, errlen, nullptr, nullptr);
    }
}

// apply_Q_thomas (thomas.cpp:128-160) of one field along `axis`.
int ref_apply_q_thomas(int dim, int n, double tau, double kappa, double q, int family, int ell,
                       int axis, const double* in, double* out, char* err, int errlen) {
    try {
        const Grid g = unit_box_grid(dim, n + 1);
        const auto op = build_operator(g, static_cast<Axis>(axis), kappa, q);
        const auto pay = build_thomas_payload(op, tau, scheme_by_family(family ? PadeFamily::P04 : PadeFamily::P02));
        const Field r = apply_Q_thomas(pay, ell, tau, field_from(g, in), static_cast<Axis>(axis));
        std::memcpy(out, r.data(), r.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return map_exc(e, err, errlen, nullptr, nullptr);
    }
}

#ifdef REF_HAS_HARNESS
// The reference study harness (harness.cpp:305-362): run_convergence writes
// <out>/convergence_*.csv, a manifest and, for problems without a closed form,
// the ETRJ reference-trajectory cache <out>/references/*.traj.  Used to make
// golden trajectory/CSV fixtures (tests/golden/make_golden_harness.py).
int ref_run_convergence(const char* problem, int m, const int* Ns, int nN, int family, int backend,
                        int coarse, double T, const char* out, double* E, char* err, int errlen) {
    try {
        RunConfig cfg;
        cfg.problem = problem;
        cfg.m = m;
        cfg.Ns.assign(Ns, Ns + nN);
        cfg.scheme = family ? PadeFamily::P04 : PadeFamily::P02;
        cfg.backend = static_cast<BackendKind>(backend);
        cfg.coarse = coarse;
        cfg.T = T;
        cfg.out = out;
        const auto rep = run_convergence(cfg);
        for (std::size_t i = 0; i < rep.rows.size(); ++i) E[i] = rep.rows[i].E;
        return 0;
    } catch (const std::exception& e) {
        return map_exc(e, err, errlen, nullptr, nullptr);
    }
}
#endif

}  // extern "C"
