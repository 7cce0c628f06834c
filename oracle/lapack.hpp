// TEST INFRASTRUCTURE ONLY — part of the CPU oracle (see oracle/README.md).
// Fortran LAPACK/BLAS entry points exported (scipy_-prefixed, 32-bit ints) by
// scipy's bundled OpenBLAS 0.3.30 (scipy.libs/libscipy_openblas-*.so). They
// stand in for the Eigen3 kernels the reference calls.
#pragma once
#include <complex>
#include <cstddef>

using lapack_int = int;
using zcomplex = std::complex<double>;

extern "C" {
void scipy_dgemm_(const char* ta, const char* tb, const lapack_int* m, const lapack_int* n,
                  const lapack_int* k, const double* alpha, const double* a, const lapack_int* lda,
                  const double* b, const lapack_int* ldb, const double* beta, double* c,
                  const lapack_int* ldc, size_t, size_t);
void scipy_zgemm_(const char* ta, const char* tb, const lapack_int* m, const lapack_int* n,
                  const lapack_int* k, const zcomplex* alpha, const zcomplex* a,
                  const lapack_int* lda, const zcomplex* b, const lapack_int* ldb,
                  const zcomplex* beta, zcomplex* c, const lapack_int* ldc, size_t, size_t);
void scipy_dtrsm_(const char* side, const char* uplo, const char* ta, const char* diag,
                  const lapack_int* m, const lapack_int* n, const double* alpha, const double* a,
                  const lapack_int* lda, double* b, const lapack_int* ldb, size_t, size_t, size_t,
                  size_t);
void scipy_ztrsm_(const char* side, const char* uplo, const char* ta, const char* diag,
                  const lapack_int* m, const lapack_int* n, const zcomplex* alpha,
                  const zcomplex* a, const lapack_int* lda, zcomplex* b, const lapack_int* ldb,
                  size_t, size_t, size_t, size_t);
void scipy_dsyevd_(const char* jobz, const char* uplo, const lapack_int* n, double* a,
                   const lapack_int* lda, double* w, double* work, const lapack_int* lwork,
                   lapack_int* iwork, const lapack_int* liwork, lapack_int* info, size_t, size_t);
void scipy_dgeqrf_(const lapack_int* m, const lapack_int* n, double* a, const lapack_int* lda,
                   double* tau, double* work, const lapack_int* lwork, lapack_int* info);
void scipy_dgeqp3_(const lapack_int* m, const lapack_int* n, double* a, const lapack_int* lda,
                   lapack_int* jpvt, double* tau, double* work, const lapack_int* lwork,
                   lapack_int* info);
void scipy_dorgqr_(const lapack_int* m, const lapack_int* n, const lapack_int* k, double* a,
                   const lapack_int* lda, const double* tau, double* work,
                   const lapack_int* lwork, lapack_int* info);
void scipy_openblas_set_num_threads(int);
int scipy_openblas_get_num_threads(void);
}
