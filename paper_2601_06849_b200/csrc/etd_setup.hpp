// Host-side one-time setup for the ETD2RK-DS spectral step (may stay on the
// host per BASELINE north_star): directional operators, closed-form Dirichlet
// eigensystems, Pade pole/residue sets and the diagonal "d-vectors".
#pragma once
#include <array>
#include <complex>
#include <stdexcept>
#include <cstddef>
#include <string>
#include <vector>

namespace etd {

struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NumericsError : std::runtime_error { using std::runtime_error::runtime_error; };
// errors.hpp:28 MemoryGuardError: the plan's device memory does not fit the cap / the device
struct MemoryGuardError : std::runtime_error { using std::runtime_error::runtime_error; };

// Toeplitz tridiagonal factor of kappa*(-Laplacian) + q along one axis
// (reference operators.cpp:11-34): diag = (2k + (q/dim) h^2)/h^2, off = -k/h^2.
struct AxisOperator {
    int n = 0;
    double h = 0.0, diag = 0.0, off = 0.0;
};
AxisOperator axis_operator(int n, double low, double high, int dim, double kappa, double q);

// Closed-form eigensystem (reference operators.cpp:36-56):
//   lambda_k = diag + 2 off cos(theta_k),  P(i,k) = sqrt(2/(n+1)) sin((i+1) theta_k),
//   theta_k = (k+1) pi/(n+1).  P returned column-major (P[k*n+i] = P(i,k)).
void eigensystem(const AxisOperator& op, std::vector<double>& P, std::vector<double>& lambda);

// Pole/residue terms of the three rational weights (reference rational.cpp:133-177).
struct PoleResidue { std::complex<double> pole, residue; };
struct PadeScheme { int family = 0; std::array<std::vector<PoleResidue>, 3> terms; };
PadeScheme pade_scheme(int family);

// d_k = sum_l Re(r_l / (tau*lambda_k - s_l)) — half of Q_ell(tau lambda_k)
// (reference rational.cpp:187-198).
std::vector<double> dvector(const std::vector<double>& lambda, double tau, const PadeScheme& s,
                            int ell);

// Thomas factors of one pole (reference thomas.cpp:14-29 factor_pole): LU of the
// Toeplitz tridiagonal with diagonal c and off-diagonals e, no pivoting,
// mul_i = e / piv_{i-1}, piv_i = c - mul_i e; inv_i = 1 / piv_i (thomas.cpp:70,76).
// NumericsError on a pivot below 1e-30 in magnitude.
struct ThomasPole { std::vector<std::complex<double>> mul, piv, inv; };
ThomasPole thomas_factor(int n, std::complex<double> c, std::complex<double> e);

// Exact-exponential multipliers (reference stepper.cpp:162-170, 276-292):
// e^{-tau lambda_k}; tau phi_1(tau lambda_k) (which = 1) or tau phi_2 (which = 2),
// phi with the reference's series branch below x = 1e-4.
double phi1(double x);
double phi2(double x);
std::vector<double> exp_multipliers(const std::vector<double>& lambda, double tau);
std::vector<double> phi_multipliers(const std::vector<double>& lambda, double tau, int which);

// Seeded initial conditions for BASELINE configs.
void fill_config_ic(int config, unsigned long long seed, int species, int n, int z0, int z1,
                    double* out);

}  // namespace etd
