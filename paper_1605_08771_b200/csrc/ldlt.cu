// Complex-symmetric LDL^T of F = z I - A without interchanges (SURVEY.md
// §8(f)3: "complex-symmetric LDL^T as a ~2x flop cut", opt-in).
//
// Why no pivoting is safe here: A is real symmetric and Im z > 0, so
// Im(F) = Im(z) I is positive definite. -iF then has a positive definite
// Hermitian part, a property every Schur complement inherits, so each pivot
// d_j of the elimination satisfies |d_j| >= Im d_j >= Im z > 0: the
// factorization exists for every node and no pivot is smaller than Im z.
//
// The factor is stored exactly like the partial-pivot LU's (unit-lower L
// below the diagonal, U = D L^T on and above it, identity permutation), so
// the blocked DMMA solves of the LU path run on it unchanged. Only the lower
// trapezoid of each trailing update is computed (launch_zgemm_sub_lower):
// 4/3 n^3 complex flops per node where the LU needs 8/3 n^3.
//
// Per 64-column panel j at k = 64 j (capi.cu factor_group_ldlt):
//   ldlt_panel   A_kk = L_kk D_k L_kk^T in shared memory; writes L_kk, D_k,
//                U_kk = D_k L_kk^T, L_kk^{-1} (solves) and L_kk^{-T} (scratch)
//   zgemm SET    W = A[k+64:, k:k+64] L_kk^{-T}               (DMMA, in place)
//   ldlt_split   L[k+64:, panel] = W D_k^{-1},  U[panel, k+64:] = W^T
#include "common.cuh"
#include "kernels.hpp"

namespace fl {

namespace {

constexpr int LW = FL_TILE;  // 64

struct LdltShared {
    double Lr[LW][LW + 1];  // L (strict lower) and D, after the elimination
    double Li[LW][LW + 1];
    double cr[2][LW], ci[2][LW];  // broadcast column (elimination) / row (inverse)
};

// One CTA per node, 256 threads: thread (i = tid & 63, q = tid >> 6) keeps
// row i's entries of the columns k = q + 4m (m < 16) in registers. Each
// elimination step and each substitution step is one CTA barrier: the owners
// of column j (row r) publish it in a double-buffered shared vector, then
// every thread updates its 16 entries from registers.
__global__ void __launch_bounds__(256) ldlt_panel_kernel(ZBatch F, int k0, ZBatch Inv, double* ltr,
                                                         double* lti, long lt_stride) {
    extern __shared__ __align__(16) unsigned char raw[];
    LdltShared& sh = *reinterpret_cast<LdltShared*>(raw);
    constexpr int NM = LW / 4;
    const int b = blockIdx.x;
    const int tid = threadIdx.x;
    const int i = tid & (LW - 1), q = tid >> 6;
    double* Fr = F.re + b * F.stride;
    double* Fi = F.im + b * F.stride;
    // the diagonal block's lower triangle, mirrored (the trailing updates
    // computed only the lower trapezoid: the upper part is stale)
    double ar[NM], ai[NM];
#pragma unroll
    for (int m = 0; m < NM; ++m) {
        const int k = q + 4 * m;
        const long o = i >= k ? (long)(k0 + k) * F.ld + k0 + i : (long)(k0 + i) * F.ld + k0 + k;
        ar[m] = Fr[o];
        ai[m] = Fi[o];
    }
    // right-looking elimination: c = column j of the Schur complement,
    // l_i = c_i / d_j, a_ik -= l_i c_k for i, k > j -- the partial-pivot LU's
    // update a_ik -= l_ij u_jk with u_jk = a_kj
    // (j = 4 mj + qj with mj unrolled: the published entry ar[mj] has a
    // static index, so the row stays in registers)
#pragma unroll
    for (int mj = 0; mj < NM; ++mj) {
#pragma unroll 1
        for (int qj = 0; qj < 4; ++qj) {
            const int j = 4 * mj + qj;
            if (j == LW - 1) break;
            const int buf = j & 1;
            if (q == qj) {
                sh.cr[buf][i] = ar[mj];
                sh.ci[buf][i] = ai[mj];
            }
            __syncthreads();
            if (i > j) {
                // 1/d = conj(d) / |d|^2: one reciprocal on the step's critical
                // path (|d| >= Im z, so no scaling is needed)
                const double dr = sh.cr[buf][j], di = sh.ci[buf][j];
                const double s2 = 1.0 / (dr * dr + di * di);
                const cplx inv{dr * s2, -di * s2};
                const cplx l = cmul(cplx{sh.cr[buf][i], sh.ci[buf][i]}, inv);
#pragma unroll
                for (int m = 0; m < NM; ++m) {
                    const int k = q + 4 * m;
                    if (k > j) {
                        const double cr = sh.cr[buf][k], ci = sh.ci[buf][k];
                        ar[m] -= l.re * cr - l.im * ci;
                        ai[m] -= l.re * ci + l.im * cr;
                    } else if (k == j) {
                        ar[m] = l.re;
                        ai[m] = l.im;
                    }
                }
            }
        }
    }
#pragma unroll
    for (int m = 0; m < NM; ++m) {
        const int k = q + 4 * m;
        if (i >= k) {
            sh.Lr[i][k] = ar[m];
            sh.Li[i][k] = ai[m];
        }
    }
    __syncthreads();
    // X = L^{-1} (unit lower), thread (i, q) holding X[i][q + 4m]: row r is
    // final after step r - 1; its owners publish it, rows below subtract
    // L[i][r] X[r][:] (only columns k <= r are non-zero)
    double xr[NM], xi[NM];
#pragma unroll
    for (int m = 0; m < NM; ++m) {
        xr[m] = (q + 4 * m == i) ? 1.0 : 0.0;
        xi[m] = 0.0;
    }
#pragma unroll 1
    for (int r = 0; r < LW - 1; ++r) {
        const int buf = r & 1;
        if (i == r) {
#pragma unroll
            for (int m = 0; m < NM; ++m) {
                sh.cr[buf][q + 4 * m] = xr[m];
                sh.ci[buf][q + 4 * m] = xi[m];
            }
        }
        __syncthreads();
        if (i > r) {
            const cplx l{sh.Lr[i][r], sh.Li[i][r]};
#pragma unroll
            for (int m = 0; m < NM; ++m) {
                const int k = q + 4 * m;
                if (k <= r) {
                    const double cr = sh.cr[buf][k], ci = sh.ci[buf][k];
                    xr[m] -= l.re * cr - l.im * ci;
                    xi[m] -= l.re * ci + l.im * cr;
                }
            }
        }
    }
    double* Ir = Inv.re + b * Inv.stride + (long)(k0 / LW) * LW * LW;
    double* Ii = Inv.im + b * Inv.stride + (long)(k0 / LW) * LW * LW;
    double* Tr = ltr + b * lt_stride;
    double* Ti = lti + b * lt_stride;
#pragma unroll
    for (int m = 0; m < NM; ++m) {
        const int k = q + 4 * m;
        Ir[(long)k * LW + i] = xr[m];  // L^{-1}, column-major ld 64
        Ii[(long)k * LW + i] = xi[m];
        Tr[(long)i * LW + k] = xr[m];  // L^{-T}
        Ti[(long)i * LW + k] = xi[m];
    }
    // the factor's diagonal block: L below, D on, U = D L^T above the diagonal
    for (int e = tid; e < LW * LW; e += 256) {
        const int r = e & (LW - 1), c = e >> 6;
        const long o = (long)(k0 + c) * F.ld + k0 + r;
        if (r >= c) {
            Fr[o] = sh.Lr[r][c];
            Fi[o] = sh.Li[r][c];
        } else {  // U_rc = d_r l_cr
            const cplx u = cmul(cplx{sh.Lr[r][r], sh.Li[r][r]}, cplx{sh.Lr[c][r], sh.Li[c][r]});
            Fr[o] = u.re;
            Fi[o] = u.im;
        }
    }
}

struct SplitShared {
    double wr[LW][LW + 1];
    double wi[LW][LW + 1];
    double dr[LW], di[LW];
};

// Tile t of W = F[r0 + 64 t : +64, k0 : k0 + 64]:
//   F[rows, k0 : k0+64] = W D^{-1}  (L)   and   F[k0 : k0+64, rows] = W^T  (U).
__global__ void __launch_bounds__(256) ldlt_split_kernel(ZBatch F, int k0, int r0) {
    extern __shared__ __align__(16) unsigned char raw[];
    SplitShared& sh = *reinterpret_cast<SplitShared*>(raw);
    const int b = blockIdx.y;
    const int r = r0 + blockIdx.x * LW;
    const int tid = threadIdx.x;
    double* Fr = F.re + b * F.stride;
    double* Fi = F.im + b * F.stride;
    if (tid < LW) {
        const long o = (long)(k0 + tid) * F.ld + k0 + tid;
        const cplx inv = crecip(cplx{Fr[o], Fi[o]});
        sh.dr[tid] = inv.re;
        sh.di[tid] = inv.im;
    }
    for (int e = tid; e < LW * LW; e += 256) {
        const int i = e & (LW - 1), c = e >> 6;
        const long o = (long)(k0 + c) * F.ld + r + i;
        sh.wr[i][c] = Fr[o];
        sh.wi[i][c] = Fi[o];
    }
    __syncthreads();
    for (int e = tid; e < LW * LW; e += 256) {
        const int i = e & (LW - 1), c = e >> 6;
        const cplx l = cmul(cplx{sh.wr[i][c], sh.wi[i][c]}, cplx{sh.dr[c], sh.di[c]});
        const long o = (long)(k0 + c) * F.ld + r + i;
        Fr[o] = l.re;
        Fi[o] = l.im;
    }
    for (int e = tid; e < LW * LW; e += 256) {
        const int c = e & (LW - 1), i = e >> 6;
        const long o = (long)(r + i) * F.ld + k0 + c;
        Fr[o] = sh.wr[i][c];
        Fi[o] = sh.wi[i][c];
    }
}

__global__ void iota_perm_kernel(int* perm, int N) {
    int* p = perm + (long)blockIdx.y * N;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) p[i] = i;
}

}  // namespace

void launch_ldlt_panel(ZBatch F, int k0, ZBatch Inv, double* ltr, double* lti, long lt_stride,
                       int batch, cudaStream_t s) {
    const size_t sm = sizeof(LdltShared);
    ensure_smem((const void*)ldlt_panel_kernel, sm);
    ldlt_panel_kernel<<<batch, 256, sm, s>>>(F, k0, Inv, ltr, lti, lt_stride);
}

void launch_ldlt_split(ZBatch F, int k0, int r0, int rows, int batch, cudaStream_t s) {
    if (rows <= 0) return;
    const size_t sm = sizeof(SplitShared);
    ensure_smem((const void*)ldlt_split_kernel, sm);
    ldlt_split_kernel<<<dim3(rows / LW, batch), 256, sm, s>>>(F, k0, r0);
}

void launch_iota_perm(int* perm, int N, int batch, cudaStream_t s) {
    iota_perm_kernel<<<dim3((N + 255) / 256, batch), 256, 0, s>>>(perm, N);
}

}  // namespace fl
