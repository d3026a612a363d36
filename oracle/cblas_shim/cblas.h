/* Prototype-only CBLAS shim used ONLY to compile the reference's
 * proj/core/src/tensor_ops.cpp for the oracle (test infrastructure).
 * The reference needs "a CBLAS (OpenBLAS works)" (proj/README.md:27) and no
 * cblas.h is installed here.  cblas_dgemm forwards to numpy's bundled
 * OpenBLAS 0.3.30 (ILP64, symbol scipy_cblas_dgemm64_), which is present in the
 * same image on the GPU box.  Enum values follow the CBLAS standard. */
#pragma once
#ifdef __cplusplus
extern "C" {
#endif
enum CBLAS_ORDER { CblasRowMajor = 101, CblasColMajor = 102 };
enum CBLAS_TRANSPOSE { CblasNoTrans = 111, CblasTrans = 112, CblasConjTrans = 113 };
typedef enum CBLAS_ORDER CBLAS_LAYOUT;
void scipy_cblas_dgemm64_(enum CBLAS_ORDER, enum CBLAS_TRANSPOSE, enum CBLAS_TRANSPOSE,
                          long long, long long, long long, double, const double*, long long,
                          const double*, long long, double, double*, long long);
static inline void cblas_dgemm(enum CBLAS_ORDER o, enum CBLAS_TRANSPOSE ta,
                               enum CBLAS_TRANSPOSE tb, int m, int n, int k, double alpha,
                               const double* a, int lda, const double* b, int ldb,
                               double beta, double* c, int ldc) {
    scipy_cblas_dgemm64_(o, ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc);
}
#ifdef __cplusplus
}
#endif
