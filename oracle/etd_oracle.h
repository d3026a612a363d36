/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the ETD2RK-DS spectral step.
 *
 * Plain-C restatement of the reference algorithm (arXiv 2601.06849, reference
 * library `etdrd`, /root/reference/proj/core).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may call it; the product never links it.
 * Parity of this restatement is pinned against the reference itself
 * (oracle/_ref/libetdrd_ref.so built from the reference sources, see
 * tests/golden/make_golden.py and tests/test_oracle.py).
 *
 * Fields are dense FP64, x-fastest: index i + nx*(j + ny*k) (field.hpp:13-54).
 * n = interior points per axis; the reference grid has m = n+1 subintervals
 * (grid.hpp:14-16), h = 1/(n+1) on the unit box.
 */
#ifndef ETD_ORACLE_H
#define ETD_ORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

/* operators.cpp:11-34 */
void etd_o_operator(int dim, int n, double kappa, double q, double* diag, double* off);
/* operators.cpp:36-56 ; P column-major n*n: P[k*n+i] = P(i,k) */
void etd_o_spectral_factor(int n, double diag, double off, double* P, double* eig);
/* rational.cpp:133-177 ; out[(ell-1)*nterms+t][4] = pole.re, pole.im, res.re, res.im */
int etd_o_scheme(int family, double* out, int* nterms);
/* rational.cpp:187-198 */
void etd_o_dvector(int n, const double* eig, double tau, int family, int ell, double* d);
/* tensor_ops.cpp:25-52,107-119: out[..k..] = sum_i A(k,i) in[..i..], A = M or M^T */
void etd_o_contract(int nx, int ny, int nz, const double* M, int axis, int transpose,
                    const double* in, double* out);
/* tensor_ops.cpp:130-172: 2 * P diag(d_ell) P^T along `axis` */
int etd_o_apply_q(int dim, int n, double tau, double kappa, double q, int family, int ell,
                  int axis, const double* in, double* out);

/* Scalar ETD2RK-DS steps (stepper.cpp:182-257).  u (n^dim) updated in place.
 * Returns 0, or 3 on a non-finite abort with *t_abort / *step_abort set as the
 * reference's StepperAbort (stepper.cpp:18-23,191,213,227). */
int etd_o_scalar_run(int dim, int n, double tau, double kappa, double q, int family,
                     int src_kind, const double* src_params, double* u, long* n_io,
                     double* t_io, int nsteps, double* t_abort, long* step_abort);
/* Two-species steps (system_stepper.cpp:74-114; 3D with the z->y filter of
 * stepper.cpp:244-247). */
int etd_o_system_run(int dim, int n, double tau, double ku, double kv, double q, int family,
                     int src_kind, const double* src_params, double* u, double* v, long* n_io,
                     double* t_io, int nsteps, double* t_abort, long* step_abort);

/* The same with BackendKind (0 Spectral, 1 Thomas: thomas.cpp:14-160, per-pole
 * tridiagonal sweeps; the 2D Thomas step is stepper.cpp:220-225). */
int etd_o_apply_q_b(int dim, int n, double tau, double kappa, double q, int family, int backend, int ell,
                    int axis, const double* in, double* out);
int etd_o_scalar_run_b(int dim, int n, double tau, double kappa, double q, int family, int backend,
                       int src_kind, const double* src_params, double* u, long* n_io,
                       double* t_io, int nsteps, double* t_abort, long* step_abort);
int etd_o_system_run_b(int dim, int n, double tau, double ku, double kv, double q, int family, int backend,
                       int src_kind, const double* src_params, double* u, double* v, long* n_io,
                       double* t_io, int nsteps, double* t_abort, long* step_abort);

#ifdef __cplusplus
}
#endif
#endif
