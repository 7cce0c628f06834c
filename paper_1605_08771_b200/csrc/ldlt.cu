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
    double Ar[LW][LW + 1];
    double Ai[LW][LW + 1];
    double Xr[LW][LW + 1];
    double Xi[LW][LW + 1];
};

// One CTA per node. 256 threads.
__global__ void __launch_bounds__(256) ldlt_panel_kernel(ZBatch F, int k0, ZBatch Inv, double* ltr,
                                                         double* lti, long lt_stride) {
    extern __shared__ __align__(16) unsigned char raw[];
    LdltShared& sh = *reinterpret_cast<LdltShared*>(raw);
    const int b = blockIdx.x;
    const int tid = threadIdx.x;
    double* Fr = F.re + b * F.stride;
    double* Fi = F.im + b * F.stride;
    // the diagonal block's lower triangle (its upper part is stale: the
    // trailing updates compute the lower trapezoid only)
    for (int e = tid; e < LW * LW; e += 256) {
        const int i = e & (LW - 1), k = e >> 6;
        if (i >= k) {
            const long o = (long)(k0 + k) * F.ld + k0 + i;
            sh.Ar[i][k] = Fr[o];
            sh.Ai[i][k] = Fi[o];
        }
        sh.Xr[i][k] = (i == k) ? 1.0 : 0.0;
        sh.Xi[i][k] = 0.0;
    }
    __syncthreads();
    // right-looking elimination on the lower triangle: column j of the Schur
    // complement c_i = a_ij, l_i = c_i / d_j, a_ik -= l_i c_k (i >= k > j) --
    // the partial-pivot LU's update a_ik -= l_ij u_jk with u_jk = a_kj
    for (int j = 0; j < LW - 1; ++j) {
        const cplx inv = crecip(cplx{sh.Ar[j][j], sh.Ai[j][j]});
        for (int e = tid; e < LW * LW; e += 256) {
            const int i = e & (LW - 1), k = e >> 6;
            if (k > j && i >= k) {
                const cplx l = cmul(cplx{sh.Ar[i][j], sh.Ai[i][j]}, inv);
                const cplx c{sh.Ar[k][j], sh.Ai[k][j]};
                sh.Ar[i][k] -= l.re * c.re - l.im * c.im;
                sh.Ai[i][k] -= l.re * c.im + l.im * c.re;
            }
        }
        __syncthreads();
        if (tid > j && tid < LW) {
            const cplx l = cmul(cplx{sh.Ar[tid][j], sh.Ai[tid][j]}, inv);
            sh.Ar[tid][j] = l.re;
            sh.Ai[tid][j] = l.im;
        }
        __syncthreads();
    }
    // X = L^{-1} (unit lower) by forward substitution on the identity:
    // thread (col = tid & 63, q = tid >> 6) owns rows q, q + 4, ...
    const int col = tid & 63, q = tid >> 6;
    for (int r = 0; r < LW - 1; ++r) {
        const cplx x{sh.Xr[r][col], sh.Xi[r][col]};
        for (int i = r + 1 + ((q - r - 1) & 3); i < LW; i += 4) {
            const cplx l{sh.Ar[i][r], sh.Ai[i][r]};
            sh.Xr[i][col] -= l.re * x.re - l.im * x.im;
            sh.Xi[i][col] -= l.re * x.im + l.im * x.re;
        }
        __syncthreads();
    }
    double* Ir = Inv.re + b * Inv.stride + (long)(k0 / LW) * LW * LW;
    double* Ii = Inv.im + b * Inv.stride + (long)(k0 / LW) * LW * LW;
    double* Tr = ltr + b * lt_stride;
    double* Ti = lti + b * lt_stride;
    for (int e = tid; e < LW * LW; e += 256) {
        const int i = e & (LW - 1), k = e >> 6;
        const long o = (long)(k0 + k) * F.ld + k0 + i;
        double vr, vi;
        if (i >= k) {  // L (strict lower) and D
            vr = sh.Ar[i][k];
            vi = sh.Ai[i][k];
        } else {  // U_ik = d_i l_ki
            const cplx u = cmul(cplx{sh.Ar[i][i], sh.Ai[i][i]}, cplx{sh.Ar[k][i], sh.Ai[k][i]});
            vr = u.re;
            vi = u.im;
        }
        Fr[o] = vr;
        Fi[o] = vi;
        Ir[(long)k * LW + i] = sh.Xr[i][k];  // L^{-1}, column-major ld 64
        Ii[(long)k * LW + i] = sh.Xi[i][k];
        Tr[(long)k * LW + i] = sh.Xr[k][i];  // L^{-T}
        Ti[(long)k * LW + i] = sh.Xi[k][i];
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
