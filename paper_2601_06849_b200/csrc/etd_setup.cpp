// Host setup math for the ETD2RK-DS spectral step.  Fresh code; each routine
// cites the reference routine whose values it must reproduce.
#include "etd_setup.hpp"

#include <algorithm>
#include <cmath>
#include <numbers>
#include <stdexcept>
#include <thread>

namespace etd {

AxisOperator axis_operator(int n, double low, double high, int dim, double kappa, double q) {
    if (n < 1) throw ConfigError("need at least one interior point per axis");
    if (!(high > low)) throw ConfigError("upper bound must exceed lower");
    if (!(kappa > 0.0)) throw ConfigError("diffusivity must be positive");
    if (q < 0.0) throw ConfigError("linear reaction coefficient must be nonnegative");
    AxisOperator op;
    op.n = n;
    op.h = (high - low) / (n + 1);  // grid.cpp:36-37 with m = n + 1 subintervals
    const double h2 = op.h * op.h;
    op.diag = (2.0 * kappa + (q / dim) * h2) / h2;  // same expression as operators.cpp:29
    op.off = -kappa / h2;
    return op;
}

void eigensystem(const AxisOperator& op, std::vector<double>& P, std::vector<double>& lambda) {
    const int n = op.n;
    P.assign(static_cast<std::size_t>(n) * n, 0.0);
    lambda.resize(n);
    // Same closed form and evaluation order as operators.cpp:43-53 so that the
    // device operates on the reference's exact P (regenerating
    // P with a different expression costs ~7e-14 of the 1e-11 budget).
    const double scale = std::sqrt(2.0 / (n + 1));
    for (int k = 0; k < n; ++k) {
        const double theta = (k + 1) * std::numbers::pi / (n + 1);
        lambda[k] = op.diag + 2.0 * op.off * std::cos(theta);
        double* col = P.data() + static_cast<std::size_t>(k) * n;
        for (int i = 0; i < n; ++i) col[i] = scale * std::sin((i + 1) * theta);
    }
}

namespace {

using cd = std::complex<double>;

cd poly(const double* c, int len, cd x) {
    cd acc = c[0];
    for (int i = 1; i < len; ++i) acc = acc * x + c[i];
    return acc;
}

// Upper-half-plane roots of x^4 + 4x^3 + 12x^2 + 24x + 24 (the (0,4) Pade
// denominator of e^{-x}).  Simultaneous (Weierstrass) iteration followed by a
// Newton polish, the construction rational.cpp:25-62 uses.
std::array<cd, 2> p04_upper_poles() {
    static const double den[5] = {1.0, 4.0, 12.0, 24.0, 24.0};
    static const double dden[4] = {4.0, 12.0, 24.0, 24.0};
    cd z[4];
    cd w = 1.0;
    for (int k = 0; k < 4; ++k) z[k] = (w *= cd(0.4, 0.9));
    for (int it = 0; it < 200; ++it) {
        double change = 0.0;
        for (int k = 0; k < 4; ++k) {
            cd prod = 1.0;
            for (int j = 0; j < 4; ++j)
                if (j != k) prod *= z[k] - z[j];
            const cd dz = poly(den, 5, z[k]) / prod;
            z[k] -= dz;
            change = std::max(change, std::abs(dz));
        }
        if (change < 1e-13) break;
    }
    for (auto& r : z) {
        for (int it = 0; it < 8; ++it) {
            const cd d = poly(dden, 4, r);
            if (std::abs(d) == 0.0) break;
            const cd s = poly(den, 5, r) / d;
            r -= s;
            if (std::abs(s) < 1e-16 * std::abs(r)) break;
        }
        if (std::abs(poly(den, 5, r)) > 1e-10) throw NumericsError("P04 pole polish did not converge");
    }
    std::vector<cd> up;
    for (auto& r : z)
        if (r.imag() > 0.0) up.push_back(r);
    if (up.size() != 2) throw NumericsError("expected two upper-half-plane P04 poles");
    std::sort(up.begin(), up.end(), [](const cd& a, const cd& b) { return a.real() < b.real(); });
    return {up[0], up[1]};
}

}  // namespace

PadeScheme pade_scheme(int family) {
    PadeScheme s;
    s.family = family;
    if (family == 0) {
        // (0,2) Pade: denominator x^2+2x+2, pole -1+i, D'(s)=2i; numerators 2, x+2, x+1
        // (rational.cpp:133-150).
        const cd p(-1.0, 1.0);
        s.terms[0] = {{p, cd(0.0, -1.0)}};
        s.terms[1] = {{p, cd(0.5, -0.5)}};
        s.terms[2] = {{p, cd(0.5, 0.0)}};
        return s;
    }
    if (family != 1) throw ConfigError("unknown Pade family");
    // (0,4) Pade: numerators 24, x^3+4x^2+12x+24, x^3+3x^2+8x+12 over the
    // quartic; residues N(s)/D'(s) (rational.cpp:152-177).
    static const double dden[4] = {4.0, 12.0, 24.0, 24.0};
    static const double n1[1] = {24.0}, n2[4] = {1.0, 4.0, 12.0, 24.0}, n3[4] = {1.0, 3.0, 8.0, 12.0};
    const auto up = p04_upper_poles();
    for (const cd& p : up) {
        const cd dp = poly(dden, 4, p);
        s.terms[0].push_back({p, poly(n1, 1, p) / dp});
        s.terms[1].push_back({p, poly(n2, 4, p) / dp});
        s.terms[2].push_back({p, poly(n3, 4, p) / dp});
    }
    return s;
}

std::vector<double> dvector(const std::vector<double>& lambda, double tau, const PadeScheme& s,
                            int ell) {
    if (ell < 1 || ell > 3) throw ConfigError("ell must be 1, 2, or 3");
    std::vector<double> d(lambda.size());
    for (std::size_t k = 0; k < lambda.size(); ++k) {
        const double x = tau * lambda[k];
        double acc = 0.0;
        for (const auto& t : s.terms[ell - 1]) acc += (t.residue / (cd(x, 0.0) - t.pole)).real();
        d[k] = acc;
    }
    return d;
}

// stepper.cpp:162-170: series branch below 1e-4 (branches agree to 1e-12 there)
ThomasPole thomas_factor(int n, std::complex<double> c, std::complex<double> e) {
    ThomasPole f;
    f.mul.assign(n, 0.0);
    f.piv.assign(n, 0.0);
    f.inv.assign(n, 0.0);
    f.piv[0] = c;
    for (int i = 1; i < n; ++i) {
        if (std::abs(f.piv[i - 1]) < 1e-30)
            throw NumericsError("Thomas pivot underflow at row " + std::to_string(i - 1));
        f.mul[i] = e / f.piv[i - 1];
        f.piv[i] = c - f.mul[i] * e;
    }
    if (std::abs(f.piv[n - 1]) < 1e-30) throw NumericsError("Thomas pivot underflow at last row");
    for (int i = 0; i < n; ++i) f.inv[i] = 1.0 / f.piv[i];
    return f;
}

double phi1(double x) {
    if (x < 1e-4) return 1.0 - x / 2.0 + x * x / 6.0 - x * x * x / 24.0;
    return (1.0 - std::exp(-x)) / x;
}
double phi2(double x) {
    if (x < 1e-4) return 0.5 - x / 6.0 + x * x / 24.0 - x * x * x / 120.0;
    return (x - 1.0 + std::exp(-x)) / (x * x);
}
std::vector<double> exp_multipliers(const std::vector<double>& lambda, double tau) {
    std::vector<double> v(lambda.size());
    for (std::size_t k = 0; k < lambda.size(); ++k) v[k] = std::exp(-tau * lambda[k]);  // stepper.cpp:279
    return v;
}
std::vector<double> phi_multipliers(const std::vector<double>& lambda, double tau, int which) {
    std::vector<double> v(lambda.size());
    for (std::size_t k = 0; k < lambda.size(); ++k) {
        const double x = tau * lambda[k];
        v[k] = tau * (which == 1 ? phi1(x) : phi2(x));                               // stepper.cpp:289-291
    }
    return v;
}

// ---- seeded inputs ---------------------------------------------------------
namespace {

inline unsigned long long mix64(unsigned long long z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
// Counter-based uniform in [0,1): value depends only on (seed, stream, idx).
inline double uniform01(unsigned long long seed, unsigned stream, unsigned long long idx) {
    const unsigned long long key = mix64(seed ^ (0xD1B54A32D192ED03ull * (stream + 1ull)));
    return static_cast<double>(mix64(key + idx) >> 11) * 0x1.0p-53;
}
inline double normal(unsigned long long seed, unsigned stream, unsigned long long idx) {
    const double u1 = uniform01(seed, stream, 2 * idx), u2 = uniform01(seed, stream, 2 * idx + 1);
    return std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(2.0 * std::numbers::pi * u2);
}

template <class F>
void parallel_for(int lo, int hi, F&& f) {
    const int nt = std::max(1, std::min<int>(std::thread::hardware_concurrency(), hi - lo));
    if (nt <= 1 || hi - lo < 2) {
        for (int z = lo; z < hi; ++z) f(z);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            for (int z = lo + t; z < hi; z += nt) f(z);
        });
    for (auto& x : th) x.join();
}

}  // namespace

void fill_config_ic(int config, unsigned long long seed, int species, int n, int z0, int z1,
                    double* out) {
    if (config < 0 || config > 4) throw ConfigError("config must be 0..4");
    const int dim = config <= 1 ? 2 : 3;
    if (dim == 2) { z0 = 0; z1 = 1; }
    if (z0 < 0 || z1 > (dim == 3 ? n : 1) || z0 >= z1) throw ConfigError("bad slab range");
    const double h = 1.0 / (n + 1), pi = std::numbers::pi;
    const std::size_t plane = static_cast<std::size_t>(n) * n;
    if (config >= 3) {
        // u0 = (0.5 + 0.1 N(0,1)) S, v0 = 0.1 N(0,1) S, S = prod sin(pi x_a), i.i.d. per point
        std::vector<double> s1(n);
        for (int i = 0; i < n; ++i) s1[i] = std::sin(pi * ((i + 1) * h));
        parallel_for(z0, z1, [&](int k) {
            for (int j = 0; j < n; ++j)
                for (int i = 0; i < n; ++i) {
                    const unsigned long long g = i + static_cast<unsigned long long>(n) * (j + static_cast<unsigned long long>(n) * k);
                    const double S = s1[i] * s1[j] * s1[k];
                    const double r = normal(seed, species == 0 ? 2u : 3u, g);
                    out[(k - z0) * plane + static_cast<std::size_t>(j) * n + i] =
                        species == 0 ? (0.5 + 0.1 * r) * S : (0.1 * r) * S;
                }
        });
        return;
    }
    if (species != 0) throw ConfigError("configs 0-2 are scalar");
    const int K = config == 0 ? 8 : config == 1 ? 32 : 6;
    const double amp = config == 2 ? 0.05 : 0.1;
    // sine tables s[m][i] = sin(m pi x_i), m = 1..K
    std::vector<double> s(static_cast<std::size_t>(K + 1) * n);
    for (int m = 1; m <= K; ++m)
        for (int i = 0; i < n; ++i) s[static_cast<std::size_t>(m) * n + i] = std::sin(m * pi * ((i + 1) * h));
    auto S = [&](int m, int i) { return s[static_cast<std::size_t>(m) * n + i]; };
    if (dim == 2) {
        // c_kl ~ U[-1,1], index (k-1) + K (l-1)
        std::vector<double> A(static_cast<std::size_t>(K) * n, 0.0);  // A[l][i] = sum_k c_kl s_k(x_i)
        for (int l = 1; l <= K; ++l)
            for (int i = 0; i < n; ++i) {
                double acc = 0.0;
                for (int k = 1; k <= K; ++k)
                    acc += (2.0 * uniform01(seed, 1, (k - 1) + static_cast<unsigned long long>(K) * (l - 1)) - 1.0) * S(k, i);
                A[static_cast<std::size_t>(l - 1) * n + i] = acc;
            }
        parallel_for(0, n, [&](int j) {
            for (int i = 0; i < n; ++i) {
                double acc = 0.0;
                for (int l = 1; l <= K; ++l) acc += A[static_cast<std::size_t>(l - 1) * n + i] * S(l, j);
                out[static_cast<std::size_t>(j) * n + i] = S(1, i) * S(1, j) + amp * acc;
            }
        });
        return;
    }
    // 3D: c_klm ~ U[-1,1], index (k-1) + K((l-1) + K(m-1))
    std::vector<double> B(static_cast<std::size_t>(K) * K * n, 0.0);  // B[m][l][i]
    for (int m = 1; m <= K; ++m)
        for (int l = 1; l <= K; ++l)
            for (int i = 0; i < n; ++i) {
                double acc = 0.0;
                for (int k = 1; k <= K; ++k)
                    acc += (2.0 * uniform01(seed, 1, (k - 1) + static_cast<unsigned long long>(K) * ((l - 1) + static_cast<unsigned long long>(K) * (m - 1))) - 1.0) * S(k, i);
                B[(static_cast<std::size_t>(m - 1) * K + (l - 1)) * n + i] = acc;
            }
    parallel_for(z0, z1, [&](int kz) {
        std::vector<double> Cm(K);
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                double acc = 0.0;
                for (int m = 1; m <= K; ++m) {
                    double c = 0.0;
                    for (int l = 1; l <= K; ++l) c += B[(static_cast<std::size_t>(m - 1) * K + (l - 1)) * n + i] * S(l, j);
                    acc += c * S(m, kz);
                }
                out[(kz - z0) * plane + static_cast<std::size_t>(j) * n + i] = S(1, i) * S(1, j) * S(1, kz) + amp * acc;
            }
    });
}

}  // namespace etd
