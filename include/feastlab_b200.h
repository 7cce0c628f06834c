/*
 * feastlab_b200.h — the C ABI of the B200-native FEAST filter hot path.
 *
 * The reference (feastlab, /root/reference/proj) has no FFI; its public
 * interface is C++ over Eigen. This header is the thin C boundary that the
 * drop-in C++ layer (include/feastlab/ headers, same names and options as
 * the headers in proj/include/feastlab/) and foreign callers (Python ctypes in
 * paper_1605_08771_b200/) bind. Every entry point below names the reference
 * interface it replaces.
 *
 * Conventions
 *   - Column-major fp64, explicit leading dimensions. No complex numbers cross
 *     the ABI except in the NodeFactorization test hook (interleaved re,im).
 *   - Every function returns an fl_status; on failure *err (may be NULL) holds
 *     the payload of the reference exception it stands for.
 *   - loc = FL_HOST: pointer is host memory; FL_DEVICE: pointer is device
 *     memory on the context's GPU (cudaMalloc / torch), ordered on the
 *     context stream.
 *   - Handles (fl_ctx, fl_matrix, fl_block, fl_filter) are not thread-safe;
 *     calls on one context are serialised by an internal mutex, so concurrent
 *     solves (CLI `compare` cells, proj/tools/feastlab_cli.cpp:290-292) must
 *     use one context each or accept serialisation.
 *   - Not a CPU fallback: without a CUDA device every compute entry returns
 *     FL_CUDA.
 */
#ifndef FEASTLAB_B200_H
#define FEASTLAB_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; the C++ layer maps them back to the reference exception types */
enum fl_status {
  FL_OK = 0,
  FL_INVALID_ARGUMENT = 1, /* std::invalid_argument                                  */
  FL_RUNTIME_ERROR = 2,    /* std::runtime_error                                     */
  FL_CHOLESKY = 3,         /* feastlab::CholeskyError (ritz.hpp:27-31): pivot, index */
  FL_SINGULAR_NODE = 4,    /* runtime_error of filterop.cpp:19-22: index, z          */
  FL_CUDA = 5,
  FL_NCCL = 6,
  FL_OOM = 7,
  FL_MATRIX_MARKET = 8,    /* feastlab::MatrixMarketError (matrix_market.hpp:9-16): index = line */
  FL_NOT_SYMMETRIC = 9     /* feastlab::NotSymmetricError (matrix_market.hpp:18-21): index = line */
};

enum fl_loc { FL_HOST = 0, FL_DEVICE = 1 };

typedef struct fl_err {
  int status;
  int index;     /* CholeskyError::index / singular node index     */
  double pivot;  /* CholeskyError::pivot                            */
  double z_re;   /* singular node shift                             */
  double z_im;
  char msg[512]; /* what()                                          */
} fl_err;

typedef struct fl_ctx fl_ctx;       /* device, stream, NCCL communicator, workspaces */
typedef struct fl_matrix fl_matrix; /* device-resident SymmetricMatrix               */
typedef struct fl_block fl_block;   /* device-resident n x p real block (MatrixXd)    */
typedef struct fl_filter fl_filter; /* FilterApplier state (rule, factor cache)       */
typedef struct fl_node fl_node;     /* NodeFactorization: one owned device LU factor  */

/* ------------------------------------------------------------ context */
int fl_version(void);
int fl_device_count(int* count);
/* one GPU, no collective */
int fl_ctx_create(int device, fl_ctx** out, fl_err* err);
/* rank `rank` of `nranks` (one process per GPU); contour nodes are sharded
   across the ranks and the filter sum is all-reduced over NCCL. `nccl_id` is
   the 128-byte ncclUniqueId made by fl_nccl_unique_id on rank 0. */
int fl_ctx_create_nccl(int device, const void* nccl_id, int rank, int nranks, fl_ctx** out,
                       fl_err* err);
int fl_nccl_unique_id(void* out128, fl_err* err);
/* Test hook: a context that plays rank `rank` of `nranks` for the node
   sharding only (no communicator): its filters factor and solve the rank's
   contour nodes and return the rank's partial sum, as a rank of a real clique
   does just before its all-reduce. Lets one GPU run every shard of a G-GPU job. */
int fl_ctx_create_virtual(int device, int rank, int nranks, fl_ctx** out, fl_err* err);
/* contour nodes owned by `rank` of `nranks`: [*k_begin, *k_end), contiguous,
   ascending; the shards of all ranks partition [0, n_c) */
int fl_node_shard(int n_c, int rank, int nranks, int* k_begin, int* k_end);
int fl_ctx_destroy(fl_ctx* ctx);
int fl_ctx_sync(fl_ctx* ctx, fl_err* err);
void* fl_ctx_stream(fl_ctx* ctx); /* cudaStream_t */
int fl_ctx_rank(const fl_ctx* ctx, int* rank, int* nranks);
/* number of kernels this context launched so far (instrumentation) */
long long fl_ctx_launches(const fl_ctx* ctx);
/* per-kernel-class CUDA-event timing on the context stream (instrumentation):
   classes "shift", "panel", "laswp", "trsm", "zgemm", "permute", "accumulate",
   "allreduce"; work = algorithmic flops (GEMM/TRSM) or bytes (streams). */
int fl_ctx_set_profiling(fl_ctx* ctx, int on);
/* number of contour-node chunks factored/solved concurrently (1..8, default 8) */
int fl_ctx_set_streams(fl_ctx* ctx, int n);
/* how a multi-rank context combines the per-rank partial filters into Y:
   FL_REDUCE_SUM (default): local ascending-k sum, then ncclAllReduce(sum) —
   one n x p exchange, rounding depends on the rank count;
   FL_REDUCE_ORDERED: all-gather of the per-node terms Re(w_k W_k), then every
   rank sums all n_c terms in ascending k (filterop.cpp:65-81 / SPEC.md:249) —
   n_c x n x p bytes exchanged, Y bitwise identical at every GPU count.
   Single-rank contexts ignore it. */
enum { FL_REDUCE_SUM = 0, FL_REDUCE_ORDERED = 1 };
int fl_ctx_set_reduction(fl_ctx* ctx, int mode);
/* how the filter factors each shifted matrix z_k I - A (per context; cached
   factors of the other kind are rebuilt at the next application):
   FL_FACTOR_LU (default): complex partial-pivot LU, the reference's
   Eigen::PartialPivLU (proj/src/filterop.cpp:14);
   FL_FACTOR_LDLT: complex-symmetric LDL^T without interchanges (SURVEY.md
   §8(f)3): z I - A is complex symmetric with Im(z I - A) = Im(z) I positive
   definite, so every pivot satisfies |d_j| >= Im z > 0 and no pivoting is
   needed; the trailing updates touch only the lower triangle, half the LU's
   8/3 n^3 flops. Results agree with the LU's to rounding (tests/
   test_gpu_ldlt.py), not bitwise. Env FEASTLAB_FACTOR=ldlt sets it for new
   contexts. */
enum { FL_FACTOR_LU = 0, FL_FACTOR_LDLT = 1 };
int fl_ctx_set_factorization(fl_ctx* ctx, int mode);
int fl_ctx_factorization(const fl_ctx* ctx); /* the mode in effect, -1 for NULL */
/* complex product form of the filter's DMMA GEMMs (process-wide): 1 = 3M
   (three real products per complex product, the default), 0 = 4M; mode < 0
   only queries. Returns the mode in effect. Env FEASTLAB_ZGEMM=4m|3m sets
   the initial value. */
int fl_zgemm_mode(int mode);
/* timeline of the profiled launches: out[5i] = class index (order of
   fl_ctx_profile's classes), out[5i+1] / out[5i+2] = start / end in ms,
   out[5i+3] = the launch's algorithmic work, out[5i+4] = its shape tag
   (GEMM classes: ((role*1024 + M/64)*1024 + N/64)*1024 + K/16, else 0) */
int fl_ctx_profile_dump(fl_ctx* ctx, double* out, int max_records);
/* microbenchmark of the planar-complex DMMA GEMM (instrumentation) */
int fl_debug_zgemm(fl_ctx* ctx, int M, int N, int K, int batch, int iters, double* ms_out,
                   fl_err* err);
/* the same product on operands laid out as in an LU trailing update: batch
   N x N planar factors, C = F[N-M:, N-M:N-M+Nc] -= F[N-M:, 0:K] F[0:K, ...].
   variant 0: the cp.async 3M/4M kernel; 1: the TMA-fed 3M kernel with
   precomputed sum planes. *checksum = a weighted sum of C after one product;
   maxdiff[0] = max |C_variant - C_variant0|, maxdiff[1] = max |F| (variant != 0)
   (instrumentation: compares kernel variants) */
int fl_debug_zgemm_lu(fl_ctx* ctx, int N, int M, int Nc, int K, int batch, int iters, int variant,
                      double* ms_out, double* checksum, double* maxdiff, fl_err* err);
/* weighted sums of the 64 x 64 tiles of the factors in slots [0, count)
   (instrumentation: compares factorizations across runs) */
int fl_debug_factor_tilesums(fl_filter* f, int count, double* out);
/* on != 0: the drivers' rounding-sensitive decisions (Gram-floor rank of
   orthonormalize, inside test of rayleigh_ritz) are written to stderr with their
   margins; on < 0 only queries. Returns the setting (instrumentation). */
int fl_debug_decision_log(int on);
/* cycle counts of the LU panel kernel's phases (instrumentation) */
int fl_debug_panel_profile(double* out8, int reset);
/* per-warp clock64 trace of the first on-chip panel (builds with FL_PANEL_TRACE) */
int fl_debug_panel_trace(long long* out, int max);
int fl_ctx_profile(fl_ctx* ctx, const char* cls, double* ms, double* work, long long* launches,
                   fl_err* err);

/* ------------------------------------------------------------ matrix
   SymmetricMatrix (proj/include/feastlab/matmodel.hpp:12-24): the caller has
   already symmetrised (fl_symmetric_matrix); the device copy is zero-padded.
   loc = FL_DEVICE: A may still be being written on another stream; the copy
   waits for the device first. (Device-resident X of fl_block_set /
   fl_filter_apply_raw must be complete before the call: they are ordered on
   the context stream only.) */
int fl_matrix_create(fl_ctx* ctx, const double* A, int n, int lda, int loc, fl_matrix** out,
                     fl_err* err);
int fl_matrix_destroy(fl_matrix* m);
int fl_matrix_dim(const fl_matrix* m);

/* ------------------------------------------------------------ blocks (Eigen::MatrixXd on device) */
int fl_block_create(fl_ctx* ctx, int n, int cap_cols, fl_block** out, fl_err* err);
int fl_block_destroy(fl_block* b);
int fl_block_cols(const fl_block* b);
int fl_block_rows(const fl_block* b);
/* upload p columns (p <= capacity) */
int fl_block_set(fl_block* b, const double* X, int ldx, int p, int loc, fl_err* err);
/* download all current columns */
int fl_block_get(const fl_block* b, double* X, int ldx, int loc, fl_err* err);
/* dst = src[:, idx[0..k-1]] (select_pairs gather, ritz.cpp:153-164; fill_solution) */
int fl_block_gather(fl_block* dst, const fl_block* src, const int* idx, int k, fl_err* err);
/* dst = [dst, src] (hconcat, drivers.cpp:84-94; RFEAST expansion, drivers.cpp:224-230) */
int fl_block_append(fl_block* dst, const fl_block* src, fl_err* err);
int fl_block_copy(fl_block* dst, const fl_block* src, fl_err* err);

/* ------------------------------------------------------------ filter (THE hot path)
   FilterApplier(A, rule, cache) (filterop.hpp:48-60): nodes z_k = zr+i zi and
   weights w_k in ascending k (ContourRule, contour.hpp:34-40). */
int fl_filter_create(fl_ctx* ctx, const fl_matrix* A, int n_c, const double* zr, const double* zi,
                     const double* wr, const double* wi, int cache_factorizations,
                     fl_filter** out, fl_err* err);
int fl_filter_destroy(fl_filter* f);
/* Y = sum_k Re(w_k (z_k I - A)^{-1} X), ascending k; FilterApplier::apply
   (filterop.cpp:62-84). accounting counters are incremented like
   SolveAccounting (filterop.hpp:15-18). */
int fl_filter_apply(fl_filter* f, const fl_block* X, fl_block* Y, long long* rhs_solved,
                    long long* factorizations, fl_err* err);
/* same on raw buffers (host or device, per loc) */
int fl_filter_apply_raw(fl_filter* f, const double* X, int ldx, int p, double* Y, int ldy, int loc,
                        long long* rhs_solved, long long* factorizations, fl_err* err);

/* ------------------------------------------------------------ Rayleigh-Ritz (ritz.hpp:39-57) */
/* orthonormalize (ritz.cpp:17-59); method 0 = svd (Gram), 1 = qr */
int fl_orthonormalize(fl_ctx* ctx, const fl_block* X, double drop_tol, int method, fl_block* U,
                      int* rank, fl_err* err);
/* rayleigh_ritz (ritz.cpp:83-118): host outputs vals[p], norms[p], inside[p]; V on device */
int fl_rayleigh_ritz(fl_ctx* ctx, const fl_matrix* A, const fl_block* X, double lo, double hi,
                     double* vals, fl_block* V, double* norms, unsigned char* inside, fl_err* err);
/* compute_residual_block (ritz.cpp:120-122) */
int fl_residual_block(fl_ctx* ctx, const fl_matrix* A, const fl_block* V, const double* vals,
                      fl_block* R, fl_err* err);
/* rank of X under ColPivHouseholderQR-style threshold (make_initial_guess, drivers.cpp:33-36) */
int fl_block_rank(fl_ctx* ctx, const fl_block* X, double threshold, int* rank, fl_err* err);
/* device symmetric eigensolve (SelfAdjointEigenSolver stand-in; test hook) */
int fl_sym_eig(fl_ctx* ctx, const double* M, int p, int ldm, double* vals, double* V, int ldv,
               fl_err* err);
/* NodeFactorization(A, z).solve(B) (filterop.cpp:9-32; test hook): interleaved complex */
int fl_node_solve(fl_ctx* ctx, const fl_matrix* A, double zr, double zi, const double* B, int p,
                  double* W, fl_err* err);
/* NodeFactorization(A, z, node_index) (filterop.cpp:9-24): factors z I - A once into an
   owned device factor; FL_SINGULAR_NODE (index = node_index) when a U diagonal entry is
   zero or non-finite. The factor lives until fl_node_destroy. */
int fl_node_create(fl_ctx* ctx, const fl_matrix* A, double zr, double zi, int node_index,
                   fl_node** out, fl_err* err);
/* NodeFactorization::solve (filterop.cpp:26-32): W = (z I - A)^{-1} B against the owned
   factor, B and W host n x p interleaved complex (column-major); no refactorisation */
int fl_node_factor_solve(fl_node* node, const double* B, int p, double* W, fl_err* err);
int fl_node_destroy(fl_node* node);

/* ------------------------------------------------------------ host-level entry points
   (the drop-in C++ layer, exported for foreign callers) */
typedef struct fl_solver_config { /* SolverConfig, drivers.hpp:12-24 */
  int m0;
  int n_c;
  int s;
  double tol;
  int max_iter;
  uint64_t seed;
  int orthogonalizer; /* 0 svd, 1 qr */
  double drop_tol;
  int cache_factorizations;
  int generalized_reduced;
} fl_solver_config;

typedef struct fl_trace_record { /* TraceRecord, drivers.hpp:26-32 */
  int iter;
  int subspace_dim;
  long long rhs_cumulative;
  double max_residual;
  int m_found;
} fl_trace_record;

/* feast_solve / xfeast_solve / rfeast_solve (drivers.hpp:58-69); variant 0/1/2.
   Capacities: values/norms m0, vectors n*m0 (ld n), trace max_iter,
   first_filtered n*m0 (optional, may be NULL: the first filtered block Y_1). */
int fl_solve(fl_ctx* ctx, int variant, const double* A, int n, int lda, double lo, double hi,
             const fl_solver_config* cfg, double* values, double* vectors, double* norms, int* m,
             int* converged, int* iterations, long long* rhs_solved, long long* factorizations,
             int* recovery_events, fl_trace_record* trace, int* ntrace, double* first_filtered,
             fl_err* err);
/* Concurrent independent solves on one matrix (extension, SURVEY §8(f)(2):
   search intervals / the CLI's compare cells, feastlab_cli.cpp:245-294):
   njobs jobs (variant[j], [lo[j], hi[j]], cfgs[j]) over per_device worker
   contexts on each of devices[0..ndev-1]. Per job: m[j] eigenvalues into
   values + j * ldv (ascending; ldv >= max m0), converged[j], iterations[j],
   max_residual[j] (last trace record), status[j] (FL_OK, or FL_RUNTIME_ERROR for a failed
   job: its message into errors + j * 256 when errors != NULL). */
int fl_solve_many(const int* devices, int ndev, int per_device, const double* A, int n, int lda,
                  int njobs, const int* variant, const double* lo, const double* hi,
                  const fl_solver_config* cfgs, double* values, int ldv, int* m, int* converged,
                  int* iterations, double* max_residual, int* status, char* errors, fl_err* err);
/* contour.hpp:28-56 */
int fl_gauss_legendre(int n, double* nodes, double* weights, fl_err* err);
int fl_build_contour_rule(double lo, double hi, int n_c, double* zr, double* zi, double* wr,
                          double* wi, fl_err* err);
double fl_filter_value(int n_c, const double* zr, const double* zi, const double* wr,
                       const double* wi, double lambda);
/* SymmetricMatrix ctor (matmodel.cpp:10-19) */
int fl_symmetric_matrix(const double* M, int n, int ldm, double sym_tol, double* out, fl_err* err);
/* make_initial_guess (drivers.cpp:23-38) — mt19937_64 + normal_distribution */
int fl_make_initial_guess(fl_ctx* ctx, int n, int m0, uint64_t seed, double* X, fl_err* err);
/* select_pairs ordering (ritz.cpp:124-151): chosen[0..*nchosen-1] */
int fl_select_pairs(const double* vals, const double* norms, const unsigned char* inside, int p,
                    int m0, double lo, double hi, int* chosen, int* nchosen, fl_err* err);
/* read_matrix_market (matrix_market.cpp:31-117) into a column-major host
   buffer: A == NULL queries *n only (banner + size line). Errors: FL_NOT_SYMMETRIC /
   FL_MATRIX_MARKET with err->index = the 1-based line; FL_RUNTIME_ERROR when the
   file cannot be opened. Pass the result to fl_matrix_create for the upload. */
int fl_mm_read(const char* path, int* n, double* A, int lda, fl_err* err);
/* write_matrix_market (matrix_market.cpp:119-147); format 0 = coordinate, 1 = array */
int fl_mm_write(const char* path, const double* A, int n, int lda, int format, fl_err* err);
/* seeded column-major N(0,1) / U[lo,hi) fills (fixture generation) */
void fl_gaussian_fill(double* out, long long count, uint64_t seed);
/* The orthogonal factor of generate_spectrum (proj/src/matmodel.cpp:93-105) on
   the device: Householder QR of the n x n block G (column-major, ld n; the
   seeded Gaussian fill of fl_gaussian_fill), Q = H_1 ... H_n I, every column
   negated when its largest-magnitude entry is negative. G, Q: FL_HOST or
   FL_DEVICE memory (loc_g, loc_q); Q has ld n. */
int fl_fixture_orthogonal(fl_ctx* ctx, const double* G, int n, int loc_g, double* Q, int loc_q,
                          fl_err* err);
/* assemble_matrix (proj/src/matmodel.cpp:109-118) on the device:
   A = 0.5 (M + M^T), M = Q diag(vals) Q^T. Q (ld n) in loc_q memory, vals (n)
   on the host, A (ld n; may alias Q) in loc_a memory. */
int fl_fixture_assemble(fl_ctx* ctx, const double* Q, int loc_q, const double* vals, int n,
                        double* A, int loc_a, fl_err* err);
void fl_uniform_fill(double* out, long long count, double lo, double hi, uint64_t seed);

#ifdef __cplusplus
}
#endif
#endif /* FEASTLAB_B200_H */
