// Internal launch interface of the Rayleigh-Ritz kernels (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>

#include "kernels.hpp"

namespace fl {

void launch_symmetrize(const double* M, long ldm, int p, double* S, long lds, cudaStream_t s);
void launch_set_diag(double* M, long ld, int from, int to, double v, cudaStream_t s);
void launch_col_norms(const double* X, long ldx, int n, int p, double* norms, cudaStream_t s);
void launch_col_div(double* X, long ldx, int n, int p, const double* d, cudaStream_t s);
void launch_residual(const double* AV, long ldav, const double* V, long ldv, int n, int p,
                     const double* lam, double* R, long ldr, cudaStream_t s);
void launch_gather_cols(const double* src, long lds, int n, const int* idx, int k, int kpad,
                        double* dst, long ldd, cudaStream_t s);
// In-place blocked Cholesky of the P x P matrix B (identity-padded beyond p);
// info_dev -> {int index (-1 ok), double pivot}.
void launch_cholesky(double* B, long ld, int p, int P, void* info_dev, cudaStream_t s);
void launch_tril(double* B, long ld, int P, cudaStream_t s);
void launch_trsm_lower(const double* L, long ldl, int P, double* X, long ldx, int ncols, bool trans,
                       cudaStream_t s);
void launch_fro2(const double* A, long lda, int p, double* out_dev, cudaStream_t s);
// Symmetric eigensolve of the p x p matrix A (destroyed; work same shape):
// ascending vals[p], eigenvectors Vout (ld ldo); V is scratch (ld ldv).
int jacobi_eig(double* A, long lda, int p, double fro, double* work, double* V, long ldv,
               double* vals, double* Vout, long ldo, int* scratch_int, unsigned long long* counters,
               int max_sweeps, cudaStream_t s);

// Block-Jacobi symmetric eigensolve of the p x p matrix A (ld lda, left
// unchanged): P = round_up(p, 64); W, V are P x P (ld P) scratch, Qbuf holds
// P x 64 doubles; ascending vals[p] and eigenvectors Vout (ld ldo). Host-driven
// sweeps (one stream synchronisation per sweep via the pinned h_counter).
int block_jacobi_eig(const double* A, long lda, int p, int P, double fro, double* W, double* V,
                     double* Qbuf, double* vals, double* Vout, long ldo,
                     unsigned long long* counters, unsigned long long* h_counter, int max_sweeps,
                     int* sweeps_out, cudaStream_t s);

// In-place column-pivoted Householder QR (dgeqp3 semantics) of the n x p matrix
// A; tau[min(n,p)], jpvt[p], norm scratch vn1/vn2[p]. Returns 0 on success.
int launch_qr(double* A, long lda, int n, int p, double* tau, int* jpvt, double* vn1, double* vn2,
              cudaStream_t s);
// Q[:, 0:r] of the reflectors left in A by launch_qr.
int launch_orgqr(const double* A, long lda, const double* tau, int n, int r, double* Q, long ldq,
                 cudaStream_t s);

// Fixture generation on the device (fixture.cu; proj/src/matmodel.cpp:93-119).
int fixture_householder_q(double* A, int N, double* Q, double* V, double* W, double* W2, double* G,
                          double* T, double* tau, cudaStream_t s);
void fixture_sign_normalize(double* Q, long ld, int n, cudaStream_t s);
void fixture_assemble(const double* Q, const double* vals, int N, int n, double* B, double* M,
                      double* A, cudaStream_t s);

}  // namespace fl
