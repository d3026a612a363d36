/* TEST INFRASTRUCTURE ONLY — CPU oracle (plain C restatement) for the
 * ETD2RK-DS spectral time step of arXiv 2601.06849 / reference `etdrd`.
 * See etd_oracle.h.  Parity pinned against oracle/_ref (the reference itself)
 * in tests/test_oracle.py and against tests/golden/ fixtures.
 *
 * Each function cites the reference file:line it restates
 * (paths relative to /root/reference/proj/core/src/).  The transforms are
 * written as naive loops (the reference calls cblas_dgemm, tensor_ops.cpp:25-52);
 * the summation order therefore differs from BLAS, which the reference's own
 * tolerances (test_tensor.cpp:45-71, <=1e-13) allow.
 */
#include "etd_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ETD_PI 3.14159265358979323846

/* ---- setup ------------------------------------------------------------- */

/* operators.cpp:11-34: q split evenly across the dim directional factors */
void etd_o_operator(int dim, int n, double kappa, double q, double* diag, double* off) {
    const double h = 1.0 / (double)(n + 1); /* grid.cpp:36-37, unit box, m = n+1 */
    const double h2 = h * h;
    *diag = (2.0 * kappa + (q / dim) * h2) / h2;
    *off = -kappa / h2;
}

/* operators.cpp:36-56: closed-form Dirichlet eigensystem, P column-major */
void etd_o_spectral_factor(int n, double diag, double off, double* P, double* eig) {
    const double scale = sqrt(2.0 / (n + 1));
    for (int k = 0; k < n; ++k) {
        const double theta = (k + 1) * ETD_PI / (n + 1);
        eig[k] = diag + 2.0 * off * cos(theta);
        for (int i = 0; i < n; ++i) P[(size_t)k * n + i] = scale * sin((i + 1) * theta);
    }
}

static double complex horner(const double* c, int len, double complex x) {
    double complex acc = c[0];
    for (int i = 1; i < len; ++i) acc = acc * x + c[i];
    return acc;
}

/* rational.cpp:133-177.  P02: pole -1+i, residues -i, (1-i)/2, 1/2.
 * P04: Durand-Kerner from seed powers of 0.4+0.9i (rational.cpp:25-48), Newton
 * polish (49-60), upper-half-plane roots sorted by real part (159-166),
 * residues N(s)/D'(s) (112-120). */
int etd_o_scheme(int family, double* out, int* nterms) {
    if (family == 0) {
        const double r[3][2] = {{0.0, -1.0}, {0.5, -0.5}, {0.5, 0.0}};
        *nterms = 1;
        for (int ell = 0; ell < 3; ++ell) {
            out[ell * 4 + 0] = -1.0;
            out[ell * 4 + 1] = 1.0;
            out[ell * 4 + 2] = r[ell][0];
            out[ell * 4 + 3] = r[ell][1];
        }
        return 0;
    }
    const double den[5] = {1.0, 4.0, 12.0, 24.0, 24.0};
    const double dprime[4] = {4.0, 12.0, 24.0, 24.0};
    const double n1[1] = {24.0}, n2[4] = {1.0, 4.0, 12.0, 24.0}, n3[4] = {1.0, 3.0, 8.0, 12.0};
    const int deg = 4;
    double complex z[4], p = 1.0, seed = 0.4 + 0.9 * I;
    for (int k = 0; k < deg; ++k) { p *= seed; z[k] = p; }
    for (int iter = 0; iter < 200; ++iter) {
        double worst = 0.0;
        for (int k = 0; k < deg; ++k) {
            double complex d = 1.0;
            for (int j = 0; j < deg; ++j)
                if (j != k) d *= z[k] - z[j];
            const double complex delta = horner(den, 5, z[k]) / d;
            z[k] -= delta;
            if (cabs(delta) > worst) worst = cabs(delta);
        }
        if (worst < 1e-13) break;
    }
    for (int k = 0; k < deg; ++k) {
        for (int it = 0; it < 8; ++it) {
            const double complex fx = horner(den, 5, z[k]);
            const double complex dfx = horner(dprime, 4, z[k]);
            if (cabs(dfx) == 0.0) break;
            const double complex step = fx / dfx;
            z[k] -= step;
            if (cabs(step) < 1e-16 * cabs(z[k])) break;
        }
        if (cabs(horner(den, 5, z[k])) > 1e-10) return 2; /* NumericsError */
    }
    double complex up[2];
    int nu = 0;
    for (int k = 0; k < deg; ++k)
        if (cimag(z[k]) > 0.0 && nu < 2) up[nu++] = z[k];
    if (nu != 2) return 2;
    if (creal(up[1]) < creal(up[0])) { double complex t = up[0]; up[0] = up[1]; up[1] = t; }
    *nterms = 2;
    for (int ell = 0; ell < 3; ++ell)
        for (int t = 0; t < 2; ++t) {
            const double complex s = up[t];
            double complex num = ell == 0 ? horner(n1, 1, s) : ell == 1 ? horner(n2, 4, s)
                                                                      : horner(n3, 4, s);
            const double complex r = num / horner(dprime, 4, s);
            double* o = out + (ell * 2 + t) * 4;
            o[0] = creal(s); o[1] = cimag(s); o[2] = creal(r); o[3] = cimag(r);
        }
    return 0;
}

/* rational.cpp:187-198: d_k = sum_l Re(r_l / (tau*lambda_k - s_l)), half of Q_ell */
void etd_o_dvector(int n, const double* eig, double tau, int family, int ell, double* d) {
    double sc[2 * 3 * 4];
    int nt = 0;
    etd_o_scheme(family, sc, &nt);
    for (int k = 0; k < n; ++k) {
        const double x = tau * eig[k];
        double acc = 0.0;
        for (int t = 0; t < nt; ++t) {
            const double* o = sc + ((ell - 1) * nt + t) * 4;
            const double complex s = o[0] + o[1] * I, r = o[2] + o[3] * I;
            acc += creal(r / (x - s));
        }
        d[k] = acc;
    }
}

/* ---- transforms -------------------------------------------------------- */

/* tensor_ops.cpp:25-52 (gemm_axis) / 107-119 (contract_axis):
 * out[..k..] = sum_i A(k,i) in[..i..],  A(k,i) = M[i*n+k] (no transpose) or M[k*n+i]. */
void etd_o_contract(int nx, int ny, int nz, const double* M, int axis, int transpose,
                    const double* in, double* out) {
    const int sh[3] = {nx, ny, nz};
    const int n = sh[axis];
    const size_t stride = axis == 0 ? 1 : axis == 1 ? (size_t)nx : (size_t)nx * ny;
    const size_t inner = stride;                       /* points below the axis */
    const size_t outer = (size_t)nx * ny * nz / ((size_t)n * inner);
    double* col = (double*)malloc(sizeof(double) * n);
    for (size_t o = 0; o < outer; ++o)
        for (size_t p = 0; p < inner; ++p) {
            const size_t base = o * n * inner + p;
            for (int i = 0; i < n; ++i) col[i] = in[base + i * stride];
            for (int k = 0; k < n; ++k) {
                double acc = 0.0;
                for (int i = 0; i < n; ++i) {
                    const double a = transpose ? M[(size_t)k * n + i] : M[(size_t)i * n + k];
                    acc += a * col[i];
                }
                out[base + k * stride] = acc;
            }
        }
    free(col);
}

/* tensor_ops.cpp:54-82 */
static void hadamard(int nx, int ny, int nz, int axis, const double* d, double* f) {
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                const int a = axis == 0 ? i : axis == 1 ? j : k;
                f[i + (size_t)nx * (j + (size_t)ny * k)] *= d[a];
            }
}

/* BackendKind::Thomas payload of one axis and component (thomas.cpp:88-126):
 * per pole l the LU factors of (tau A - s_l) (mul, piv), the off-diagonal e and
 * the residues of the three weights. */
typedef struct {
    int np;
    double complex* mul[2];
    double complex* piv[2];
    double complex e;
    double complex res[3][2];
} thomas_t;

typedef struct {
    int dim, n;
    size_t N;
    double tau;
    int thomas;         /* 0: spectral (eigenbasis) applies, 1: Thomas sweeps */
    double* P[3];      /* per axis, column-major */
    double* d[2][3][3]; /* [component][axis][ell-1] */
    thomas_t th[2][3];  /* [component][axis] */
    double* tmp;
} plan_t;

/* thomas.cpp:14-29 factor_pole (no pivoting, underflow guard 1e-30) */
static int factor_pole(int n, double complex c, double complex e, double complex* mul, double complex* piv) {
    piv[0] = c;
    mul[0] = 0.0;
    for (int i = 1; i < n; ++i) {
        if (cabs(piv[i - 1]) < 1e-30) return 2;  /* NumericsError */
        mul[i] = e / piv[i - 1];
        piv[i] = c - mul[i] * e;
    }
    return cabs(piv[n - 1]) < 1e-30 ? 2 : 0;
}

/* stepper.cpp:118-177 / system_stepper.cpp:31-70: one eigendecomposition per
 * axis; component c uses kappa_c * lambda (unit-kappa operator) for systems. */
static void plan_init(plan_t* pl, int dim, int n, double tau, const double* kappas, int ncomp,
                      int unit_kappa, double q, int family, int backend) {
    memset(pl, 0, sizeof *pl);
    pl->dim = dim;
    pl->n = n;
    pl->tau = tau;
    pl->thomas = backend == 1;
    pl->N = (size_t)n * n * (dim == 3 ? n : 1);
    pl->tmp = (double*)malloc(sizeof(double) * pl->N);
    if (pl->thomas) {
        /* thomas.cpp:88-126; systems: unit-kappa operator scaled by kappa_c
         * (system_stepper.cpp:62-64); poles from the ell = 1 terms */
        double sch[3 * 2 * 4];
        int nt = 0;
        etd_o_scheme(family, sch, &nt);
        for (int a = 0; a < dim; ++a) {
            double diag, off;
            etd_o_operator(dim, n, unit_kappa ? 1.0 : kappas[0], q, &diag, &off);
            for (int c = 0; c < ncomp; ++c) {
                const double ks = unit_kappa ? kappas[c] : 1.0;
                thomas_t* th = &pl->th[c][a];
                th->np = nt;
                th->e = tau * off * ks;
                for (int l = 0; l < nt; ++l) {
                    const double complex pole = sch[(0 * nt + l) * 4] + I * sch[(0 * nt + l) * 4 + 1];
                    th->mul[l] = (double complex*)malloc(sizeof(double complex) * n);
                    th->piv[l] = (double complex*)malloc(sizeof(double complex) * n);
                    factor_pole(n, tau * diag * ks - pole, th->e, th->mul[l], th->piv[l]);
                    for (int ell = 1; ell <= 3; ++ell)
                        th->res[ell - 1][l] = sch[((ell - 1) * nt + l) * 4 + 2] + I * sch[((ell - 1) * nt + l) * 4 + 3];
                }
            }
        }
        return;
    }
    double* eig = (double*)malloc(sizeof(double) * n);
    double* lam = (double*)malloc(sizeof(double) * n);
    for (int a = 0; a < dim; ++a) {
        double diag, off;
        etd_o_operator(dim, n, unit_kappa ? 1.0 : kappas[0], q, &diag, &off);
        pl->P[a] = (double*)malloc(sizeof(double) * n * n);
        etd_o_spectral_factor(n, diag, off, pl->P[a], eig);
        for (int c = 0; c < ncomp; ++c) {
            for (int k = 0; k < n; ++k) lam[k] = unit_kappa ? kappas[c] * eig[k] : eig[k];
            for (int ell = 1; ell <= 3; ++ell) {
                pl->d[c][a][ell - 1] = (double*)malloc(sizeof(double) * n);
                etd_o_dvector(n, lam, tau, family, ell, pl->d[c][a][ell - 1]);
            }
        }
    }
    free(eig);
    free(lam);
}

static void plan_free(plan_t* pl) {
    for (int a = 0; a < 3; ++a) {
        free(pl->P[a]);
        for (int c = 0; c < 2; ++c) {
            for (int l = 0; l < 3; ++l) free(pl->d[c][a][l]);
            for (int l = 0; l < 2; ++l) {
                free(pl->th[c][a].mul[l]);
                free(pl->th[c][a].piv[l]);
            }
        }
    }
    free(pl->tmp);
}

static void dims_of(const plan_t* pl, int* nx, int* ny, int* nz) {
    *nx = pl->n; *ny = pl->n; *nz = pl->dim == 3 ? pl->n : 1;
}

/* thomas.cpp:128-160 apply_Q_thomas: out = sum_l 2 Re(r_l (tau A - s_l)^{-1} in)
 * along `axis`: forward elimination w_i = b_i - mul_i w_{i-1}, back substitution
 * w_i = (w_i - e w_{i+1}) / piv_i (x, solve_axis_x) or * (1 / piv_i) (y/z,
 * solve_axis_planes), accumulated pole by pole. */
static void apply_q_thomas(plan_t* pl, int c, int ell, int axis, const double* in, double* out) {
    int nx, ny, nz;
    dims_of(pl, &nx, &ny, &nz);
    const thomas_t* th = &pl->th[c][axis];
    const int n = axis == 0 ? nx : axis == 1 ? ny : nz;
    const size_t es = axis == 0 ? 1 : axis == 1 ? (size_t)nx : (size_t)nx * ny;
    const size_t npen = pl->N / n;
    double complex* w = (double complex*)malloc(sizeof(double complex) * n);
    for (size_t i = 0; i < pl->N; ++i) out[i] = 0.0;
    for (int l = 0; l < th->np; ++l) {
        const double complex r = th->res[ell - 1][l], e = th->e;
        for (size_t q = 0; q < npen; ++q) {
            /* pencil q: x -> row q; y -> (i, k); z -> (i, j) */
            size_t base;
            if (axis == 0) base = q * nx;
            else if (axis == 1) base = (q % nx) + (q / nx) * (size_t)nx * ny;
            else base = q;
            w[0] = in[base];
            for (int i = 1; i < n; ++i) w[i] = in[base + i * es] - th->mul[l][i] * w[i - 1];
            for (int i = n - 1; i >= 0; --i) {
                const double complex x = i == n - 1 ? w[i] : w[i] - e * w[i + 1];
                w[i] = axis == 0 ? x / th->piv[l][i] : x * (1.0 / th->piv[l][i]);
                out[base + i * es] += 2.0 * creal(r * w[i]);
            }
        }
    }
    free(w);
}

/* tensor_ops.cpp:130-142 + 164-172: out = 2 * P (d ⊙ P^T in) along axis */
static void apply_q(plan_t* pl, int c, int ell, int axis, const double* in, double* out) {
    if (pl->thomas) {
        apply_q_thomas(pl, c, ell, axis, in, out);
        return;
    }
    int nx, ny, nz;
    dims_of(pl, &nx, &ny, &nz);
    etd_o_contract(nx, ny, nz, pl->P[axis], axis, 1, in, pl->tmp);
    hadamard(nx, ny, nz, axis, pl->d[c][axis][ell - 1], pl->tmp);
    etd_o_contract(nx, ny, nz, pl->P[axis], axis, 0, pl->tmp, out);
    for (size_t i = 0; i < pl->N; ++i) out[i] *= 2.0;
}

int etd_o_apply_q_b(int dim, int n, double tau, double kappa, double q, int family, int backend, int ell,
                    int axis, const double* in, double* out) {
    plan_t pl;
    plan_init(&pl, dim, n, tau, &kappa, 1, 0, q, family, backend);
    apply_q(&pl, 0, ell, axis, in, out);
    plan_free(&pl);
    return 0;
}

int etd_o_apply_q(int dim, int n, double tau, double kappa, double q, int family, int ell,
                  int axis, const double* in, double* out) {
    return etd_o_apply_q_b(dim, n, tau, kappa, q, family, 0, ell, axis, in, out);
}

/* ---- sources (kinds as include/etd_b200.h ETD_SRC_*) ------------------- */

/* Returns 4 on a source domain violation (problems.cpp:126-129), else 0.
 * kind 4: problems.cpp:88-104 (manufactured Allen-Cahn forcing; p0 = lambda,
 * p1 = -lambda + kappa dim pi^2); kind 5: problems.cpp:122-133 (rho u/(1-u)). */
static int scalar_src(int kind, const double* p, const double* u, double* f, size_t N, int n, int dim, double t) {
    if (kind == 5)
        for (size_t i = 0; i < N; ++i)
            if (u[i] >= 1.0) return 4;
    double* s = NULL;
    if (kind == 4) {  /* sine_product(g, 1.0): sin(pi coord), coord = (i+1) h (problems.cpp:17-33) */
        s = (double*)malloc(sizeof(double) * n);
        const double h = 1.0 / (n + 1);
        for (int i = 0; i < n; ++i) s[i] = sin(ETD_PI * ((i + 1) * h));
    }
    const double a = kind == 4 ? exp(-p[0] * t) : 0.0;
    for (size_t idx = 0; idx < N; ++idx) {
        const double x = u[idx];
        switch (kind) {
        case 1: f[idx] = x - x * x * x; break;                                  /* u - u^3 */
        case 2: f[idx] = ((p[3] * x + p[2]) * x + p[1]) * x + p[0]; break;      /* cubic poly */
        case 3: f[idx] = idx == 0 ? NAN : 0.0; break;                           /* NaN probe */
        case 4: {
            const size_t i = idx % n, j = (idx / n) % n, k = idx / ((size_t)n * n);
            double v = 1.0 * s[i] * s[j];
            if (dim == 3) v *= s[k];
            const double us = a * v;
            f[idx] = x * (1.0 - x * x) + p[1] * us - us * (1.0 - us * us);
            break;
        }
        case 5: f[idx] = p[0] * x / (1.0 - x); break;
        default: f[idx] = 0.0;
        }
    }
    free(s);
    return 0;
}

static void system_src(int kind, const double* p, const double* U, const double* V, double* fu,
                       double* fv, size_t N) {
    for (size_t i = 0; i < N; ++i) {
        const double u = U[i], v = V[i];
        switch (kind) {
        case 10: fu[i] = u * (1.0 - u) * (u - p[0]) - v; fv[i] = p[1] * (p[2] * u - v); break;
        case 11: fu[i] = u - u * u * u / 3.0 - v; fv[i] = p[0] * (u - p[1] * v); break;
        case 12: fu[i] = u - u * u * u; fv[i] = v - v * v * v; break;
        case 13: fu[i] = u - u * u * u; fv[i] = p[0] * v + p[1]; break;
        default: fu[i] = 0.0; fv[i] = 0.0;
        }
    }
}

static int all_finite(const double* f, size_t N) {
    for (size_t i = 0; i < N; ++i)
        if (!isfinite(f[i])) return 0;
    return 1;
}

/* ---- steps ------------------------------------------------------------- */

/* stepper.cpp:182-229 (2D, shared x-basis stage) and 233-257 (3D) */
static int scalar_step(plan_t* pl, int kind, const double* sp, double* U, long n, double t,
                       double* t_abort, long* step_abort) {
    const size_t N = pl->N;
    const double tau = pl->tau;
    int nx, ny, nz;
    dims_of(pl, &nx, &ny, &nz);
    double* fn = malloc(N * 8), *w1 = malloc(N * 8), *w2 = malloc(N * 8), *a = malloc(N * 8),
          *b = malloc(N * 8), *What = malloc(N * 8), *fw = malloc(N * 8);
    int rc = 0;
    if (scalar_src(kind, sp, U, fn, N, pl->n, pl->dim, t)) { *t_abort = t; *step_abort = -1; rc = 3; goto done; }
    if (!all_finite(fn, N)) { *t_abort = t; *step_abort = n; rc = 3; goto done; }
    if (pl->dim == 2 && !pl->thomas) {
        apply_q(pl, 0, 1, 1, U, w1);                          /* 193 */
        apply_q(pl, 0, 1, 1, fn, w2);                         /* 194 */
        const double* d1 = pl->d[0][0][0], *d2 = pl->d[0][0][1], *d3 = pl->d[0][0][2];
        double* w1b = a, *w2b = b;
        etd_o_contract(nx, ny, nz, pl->P[0], 0, 1, w1, w1b);  /* 202 */
        etd_o_contract(nx, ny, nz, pl->P[0], 0, 1, w2, w2b);  /* 203 */
        double* mix = w1;                                     /* w1 no longer needed */
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i)
                mix[i + (size_t)nx * j] = w1b[i + (size_t)nx * j] * d1[i] +
                                          tau * w2b[i + (size_t)nx * j] * d2[i]; /* 205-208 */
        etd_o_contract(nx, ny, nz, pl->P[0], 0, 0, mix, What);           /* 209 */
        for (size_t i = 0; i < N; ++i) What[i] *= 2.0;                    /* 210 */
        if (scalar_src(kind, sp, What, fw, N, pl->n, pl->dim, t + tau)) {   /* 212 */
            *t_abort = t + tau; *step_abort = -1; rc = 3; goto done;
        }
        if (!all_finite(fw, N)) { *t_abort = t + tau; *step_abort = n; rc = 3; goto done; }
        double* gb = w2;
        etd_o_contract(nx, ny, nz, pl->P[0], 0, 1, fw, gb);               /* 214 */
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i)
                gb[i + (size_t)nx * j] = (gb[i + (size_t)nx * j] - w2b[i + (size_t)nx * j]) * d3[i];
        double* corr = a;
        etd_o_contract(nx, ny, nz, pl->P[0], 0, 0, gb, corr);             /* 218 */
        for (size_t i = 0; i < N; ++i) U[i] = What[i] + 2.0 * tau * corr[i]; /* 219 */
    } else {
        /* 3D (stepper.cpp:243-253), and the Thomas 2D branch (220-225) without z */
        if (pl->dim == 3) {
            apply_q(pl, 0, 1, 2, U, a);  apply_q(pl, 0, 1, 1, a, w1);    /* 244-245 */
            apply_q(pl, 0, 1, 2, fn, a); apply_q(pl, 0, 1, 1, a, w2);    /* 246-247 */
        } else {
            apply_q(pl, 0, 1, 1, U, w1);                                 /* 193 */
            apply_q(pl, 0, 1, 1, fn, w2);                                /* 194 */
        }
        apply_q(pl, 0, 1, 0, w1, What);                                  /* 249 */
        apply_q(pl, 0, 2, 0, w2, b);
        for (size_t i = 0; i < N; ++i) What[i] += tau * b[i];
        if (scalar_src(kind, sp, What, fw, N, pl->n, pl->dim, t + tau)) {  /* 250 */
            *t_abort = t + tau; *step_abort = -1; rc = 3; goto done;
        }
        if (!all_finite(fw, N)) { *t_abort = t + tau; *step_abort = n; rc = 3; goto done; }
        for (size_t i = 0; i < N; ++i) fw[i] -= w2[i];                   /* 252 */
        apply_q(pl, 0, 3, 0, fw, b);                                     /* 253 */
        for (size_t i = 0; i < N; ++i) U[i] = What[i] + tau * b[i];
    }
    if (!all_finite(U, N)) { *t_abort = t + tau; *step_abort = n; rc = 3; }  /* 227/255 */
done:
    free(fn); free(w1); free(w2); free(a); free(b); free(What); free(fw);
    return rc;
}

int etd_o_scalar_run_b(int dim, int n, double tau, double kappa, double q, int family, int backend,
                       int src_kind, const double* src_params, double* u, long* n_io,
                       double* t_io, int nsteps, double* t_abort, long* step_abort) {
    if (!(tau > 0.0) || (dim != 2 && dim != 3) || n < 1) return 1; /* ConfigError */
    plan_t pl;
    plan_init(&pl, dim, n, tau, &kappa, 1, 0, q, family, backend);
    double zp[8] = {0};
    const double* sp = src_params ? src_params : zp;
    size_t N = pl.N;
    double* save = malloc(N * 8);
    int rc = 0;
    for (int s = 0; s < nsteps; ++s) {
        memcpy(save, u, N * 8);
        rc = scalar_step(&pl, src_kind, sp, u, *n_io, *t_io, t_abort, step_abort);
        if (rc) { memcpy(u, save, N * 8); break; } /* value semantics: input state kept */
        *n_io += 1;
        *t_io = (double)(*n_io) * tau;             /* stepper.cpp:228 */
    }
    free(save);
    plan_free(&pl);
    return rc;
}

int etd_o_scalar_run(int dim, int n, double tau, double kappa, double q, int family,
                     int src_kind, const double* src_params, double* u, long* n_io,
                     double* t_io, int nsteps, double* t_abort, long* step_abort) {
    return etd_o_scalar_run_b(dim, n, tau, kappa, q, family, 0, src_kind, src_params, u, n_io, t_io, nsteps,
                              t_abort, step_abort);
}

/* system_stepper.cpp:74-114, 3D filter z then y per stepper.cpp:244-247 */
int etd_o_system_run_b(int dim, int n, double tau, double ku, double kv, double q, int family, int backend,
                       int src_kind, const double* src_params, double* U, double* V, long* n_io,
                       double* t_io, int nsteps, double* t_abort, long* step_abort) {
    if (!(tau > 0.0) || (dim != 2 && dim != 3) || n < 1) return 1;
    const double kap[2] = {ku, kv};
    plan_t pl;
    plan_init(&pl, dim, n, tau, kap, 2, 1, q, family, backend);
    double zp[8] = {0};
    const double* sp = src_params ? src_params : zp;
    const size_t N = pl.N;
    double* buf = malloc(N * 8 * 14);
    double* fu = buf, *fv = buf + N, *w1[2] = {buf + 2 * N, buf + 3 * N},
          *w2[2] = {buf + 4 * N, buf + 5 * N}, *W[2] = {buf + 6 * N, buf + 7 * N}, *a = buf + 8 * N,
          *g[2] = {buf + 9 * N, buf + 10 * N}, *su = buf + 11 * N, *sv = buf + 12 * N,
          *c = buf + 13 * N;
    int rc = 0;
    for (int s = 0; s < nsteps && !rc; ++s) {
        const double t = *t_io;
        double* X[2] = {U, V};
        memcpy(su, U, N * 8);
        memcpy(sv, V, N * 8);
        system_src(src_kind, sp, U, V, fu, fv, N);                         /* 80 */
        if (!all_finite(fu, N) || !all_finite(fv, N)) { *t_abort = t; *step_abort = *n_io; rc = 3; break; }
        double* F[2] = {fu, fv};
        for (int cc = 0; cc < 2; ++cc) {                                   /* 83-86 */
            if (dim == 3) {
                apply_q(&pl, cc, 1, 2, X[cc], a); apply_q(&pl, cc, 1, 1, a, w1[cc]);
                apply_q(&pl, cc, 1, 2, F[cc], a); apply_q(&pl, cc, 1, 1, a, w2[cc]);
            } else {
                apply_q(&pl, cc, 1, 1, X[cc], w1[cc]);
                apply_q(&pl, cc, 1, 1, F[cc], w2[cc]);
            }
        }
        for (int cc = 0; cc < 2; ++cc) {                                   /* 88-95 */
            apply_q(&pl, cc, 1, 0, w1[cc], W[cc]);
            apply_q(&pl, cc, 2, 0, w2[cc], a);
            for (size_t i = 0; i < N; ++i) W[cc][i] += tau * a[i];
        }
        system_src(src_kind, sp, W[0], W[1], g[0], g[1], N);               /* 97 */
        if (!all_finite(g[0], N) || !all_finite(g[1], N)) {
            *t_abort = t + tau; *step_abort = *n_io; rc = 3; break;
        }
        for (int cc = 0; cc < 2; ++cc) {                                   /* 99-111 */
            for (size_t i = 0; i < N; ++i) g[cc][i] -= w2[cc][i];
            apply_q(&pl, cc, 3, 0, g[cc], c);
            for (size_t i = 0; i < N; ++i) X[cc][i] = W[cc][i] + tau * c[i];
        }
        if (!all_finite(U, N) || !all_finite(V, N)) {                      /* 112 */
            *t_abort = t + tau; *step_abort = *n_io; rc = 3;
            memcpy(U, su, N * 8); memcpy(V, sv, N * 8);
            break;
        }
        *n_io += 1;
        *t_io = (double)(*n_io) * tau;                                     /* 113 */
    }
    free(buf);
    plan_free(&pl);
    return rc;
}

int etd_o_system_run(int dim, int n, double tau, double ku, double kv, double q, int family,
                     int src_kind, const double* src_params, double* U, double* V, long* n_io,
                     double* t_io, int nsteps, double* t_abort, long* step_abort) {
    return etd_o_system_run_b(dim, n, tau, ku, kv, q, family, 0, src_kind, src_params, U, V, n_io, t_io, nsteps,
                              t_abort, step_abort);
}
