// Internal launch interface of the sm_100a kernels (not part of the C ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace fl {

// A kernel launch the runtime refused (bad configuration, missing attribute):
// the C ABI reports it as FL_CUDA.
struct LaunchError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
inline void launch_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw LaunchError(std::string(what) + ": " + cudaGetErrorString(e));
}

// Opt a kernel into > 48 KB dynamic shared memory once per (kernel, device).
void ensure_smem(const void* func, size_t bytes);
// Set a function attribute once per (kernel, device, attribute): the settings
// are per device, so a process driving several GPUs must set them on each.
void ensure_attr(const void* func, cudaFuncAttribute attr, int value);

// Real C = alpha op(A) op(B) + beta C. M, N multiples of 64; K multiple of 16.
struct DGemm {
    int M, N, K;
    const double* A; long lda; long strideA;
    const double* B; long ldb; long strideB;
    double* C; long ldc; long strideC;
    double alpha, beta;
};
void launch_dgemm(const DGemm& g, bool ta, bool tb, int batch, cudaStream_t s);

// Planar complex C -= A B. M, N multiples of 64; K multiple of 16.
struct ZGemm {
    int M, N, K;
    const double *Ar, *Ai; long lda; long strideA;
    const double *Br, *Bi; long ldb; long strideB;
    double *Cr, *Ci; long ldc; long strideC;
    // lower-trapezoid mode (complex-symmetric trailing updates): only the
    // 64x64 tiles (bx, by) of C with bx >= by + tri_s are computed (tri_s =
    // (column origin - row origin of C) / 64), enumerated column by column
    // on a 1-D grid (launch_zgemm_sub_lower)
    bool tri = false;
    int tri_s = 0;
    // > 0: launch order walks groups of `raster` row tiles (gemm.cu raster_tile)
    int raster = 0;
};
void launch_zgemm_sub(const ZGemm& g, int batch, cudaStream_t s);
// C -= A B on the lower trapezoid of C only (see ZGemm::tri_s)
void launch_zgemm_sub_lower(const ZGemm& g, int tri_s, int batch, cudaStream_t s);
// The TMA-fed 3M kernel for long-K trailing updates (gemm_tma.cu). Operands are
// addressed through tensor maps (make_tma_map_mk for the 64-contiguous A side,
// make_tma_map_km for the k-contiguous B side; rows multiple of 64) by element
// coordinates: A = map[a_row + ., a_col + ., a_node + z], and the precomputed
// sum planes As = Ar + Ai, Bs = Br + Bi (launch_zsum) likewise.
struct ZGemmMaps {
    CUtensorMap Ar, Ai, As, Br, Bi, Bs;
};
struct ZGemmTma {
    int M, N, K;
    int a_row, a_col, a_node;
    int as_row, as_col, as_node;
    int b_row, b_col, b_node;
    int bs_row, bs_col, bs_node;
    double *Cr, *Ci; long ldc; long strideC;
    bool tri = false;
    int tri_s = 0;
    int raster = 0;
    int rotate = 1;  // producer role rotates over the warps (gemm_tma.cu)
};
void make_tma_map_mk(CUtensorMap* m, const double* base, long rows, long cols, long ld, long stride,
                     int batch);
void make_tma_map_km(CUtensorMap* m, const double* base, long rows, long cols, long ld, long stride,
                     int batch);
void launch_zgemm_sub_tma(const ZGemmMaps& m, const ZGemmTma& g, int batch, cudaStream_t s);
// out = re + im over rows x cols (rows even), batch planes `stride` / `ostride` apart
void launch_zsum(const double* re, const double* im, long ld, long stride, double* out, long lds,
                 long ostride, int rows, int cols, int batch, cudaStream_t s);
// Complex product form of the zgemm launches: 1 = 3M (default), 0 = 4M.
int zgemm_mode();
void set_zgemm_mode(int mode);
// Planar complex C = A B (in place with B == C allowed: each CTA reads its
// whole K range before storing).
void launch_zgemm_set(const ZGemm& g, int batch, cudaStream_t s);

// A planar-complex batch of N x N factor matrices: node b's planes start at
// re + b*stride and im + b*stride, leading dimension ld (= N).
struct ZBatch {
    double* re;
    double* im;
    long ld;
    long stride;
};

// nodes per launch of the node-batched kernels (a filter has any number of
// nodes: the orchestration launches them in groups of at most kMaxNodes)
constexpr int kMaxNodes = 64;
struct NodeShifts {
    double zr[kMaxNodes];
    double zi[kMaxNodes];
};

// F_b = z_b I - A (A real N x N, zero-padded beyond n).
void launch_shift(const double* A, long lda, int N, ZBatch F, const NodeShifts& z, int batch,
                  cudaStream_t s);
// Factor panel columns [k0, k0+64) of every node (cluster kernel). ipiv[b*N + j];
// ptab[b*257 ...] receives the panel's net row permutation (count, rows, sources);
// Inv block k0/64 (see launch_trinv) receives L_kk^{-1}.
// Panels of at most `res_rows` rows (<= 4096) use the on-chip cluster panel
// (panel_res.cu, latency-optimised, whole SMs); taller ones the register-leaf
// panel that co-resides with the GEMM CTAs (throughput-optimised).
void launch_panel(ZBatch F, int N, int k0, int* ipiv, int* ptab, ZBatch Inv, int batch,
                  cudaStream_t s, int res_rows = 4096);
// Cycle counts of the panel kernel phases (node 0, rank 0, thread 0).
void panel_profile(double* out8, bool reset);
// clock64 trace of the on-chip panel (FL_PANEL_TRACE builds)
int res_panel_trace(long long* out, int max);
// Apply a panel's 64 row interchanges (ptab) to the columns [a0,a1) U [b0,b1).
void launch_laswp(ZBatch F, int a0, int a1, int b0, int b1, const int* ptab, int batch,
                  cudaStream_t s);
// Outer-block form: the composition of the np panel tables of the outer block
// at k0 (tables ptab + j * panel_stride, j < np <= 16) applied in one pass to
// the columns [a0,a1) U [b0,b1), both outside the block. cmap: N ints per node,
// identity on entry and on exit (launch_perm_identity); btab: LB_TAB ints per
// node of scratch.
constexpr int LB_MAX = 16 * 64;  // rows of the widest outer block
constexpr int LB_TAB = 1 + 3 * LB_MAX;
void launch_perm_identity(int* cmap, int N, int batch, cudaStream_t s);
void launch_laswp_block(ZBatch F, int N, int k0, int np, int a0, int a1, int b0, int b1,
                        const int* ptab, long panel_stride, int* cmap, int* btab, int batch,
                        cudaStream_t s);
// Inverses of `nblocks` consecutive 64x64 diagonal blocks starting at (r0, r0):
// unit-lower (upper=false) or upper. Block j of node b is stored at
// Inv.re/im + b*Inv.stride + (first_block + j)*4096, column-major ld 64.
void launch_trinv(ZBatch T, int r0, int nblocks, bool upper, ZBatch Inv, int first_block,
                  int batch, cudaStream_t s);
// perm[b*N + i] from the row interchanges ipiv (LAPACK-style sequence).
void launch_ipiv_to_perm(const int* ipiv, int* perm, int N, int batch, cudaStream_t s);
// W_b = complex(P_b X): Wr[i,c] = X[perm[i], c], Wi = 0 for c < P.
void launch_permute_rhs(const double* X, long ldx, int N, int P, const int* perm, ZBatch W,
                        int batch, cudaStream_t s);
// Y (+)= sum_{b ascending} Re(w_b W_b): Y = beta*Y + sum (beta in {0,1}).
void launch_accumulate(ZBatch W, int N, int P, const NodeShifts& w, int batch, double* Y, long ldy,
                       bool add_to_Y, cudaStream_t s);
// G-invariant reduction: T[b] = Re(w_b W_b) (tstride apart), then on every
// rank Y = sum over global nodes k ascending of T[slot[k]].
struct NodeSlots {
    int slot[kMaxNodes];
};
void launch_node_terms(ZBatch W, int N, int P, const NodeShifts& w, int batch, double* T,
                       long tstride, cudaStream_t s);
// Y [+]= sum_k T[slot[k]] for the nc (<= kMaxNodes) slots given, ascending
void launch_ordered_sum(const double* T, long tstride, const NodeSlots& sl, int nc, int N, int P,
                        double* Y, long ldy, bool add_to_Y, cudaStream_t s);
// Complex-symmetric LDL^T without interchanges (ldlt.cu): factor the 64x64
// diagonal block at (k0, k0) of every node (lower triangle read), write L_kk,
// D_k, U_kk = D_k L_kk^T in place, L_kk^{-1} into Inv block k0/64 and L_kk^{-T}
// (column-major ld 64) at ltr/lti + b*lt_stride.
void launch_ldlt_panel(ZBatch F, int k0, ZBatch Inv, double* ltr, double* lti, long lt_stride,
                       int batch, cudaStream_t s);
// W = F[r0 : r0+rows, k0 : k0+64] -> L = W D_k^{-1} in place, U[k0 rows, r0 : r0+rows] = W^T.
void launch_ldlt_split(ZBatch F, int k0, int r0, int rows, int batch, cudaStream_t s);
// perm[b*N + i] = i
void launch_iota_perm(int* perm, int N, int batch, cudaStream_t s);
// |U_ii| > 0 and finite for all i < n; on failure atomicMin(bad_node, offset + b).
void launch_check_diag(ZBatch F, int n, int batch, int offset, int* bad_node, cudaStream_t s);

}  // namespace fl
