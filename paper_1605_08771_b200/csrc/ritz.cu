// Rayleigh-Ritz / orthonormalisation device kernels (proj/src/ritz.cpp:17-122):
// symmetrise, blocked Cholesky with first-failing-pivot report, real 64x64
// triangular blocks, parallel cyclic Jacobi symmetric eigensolver (ascending
// output, SelfAdjointEigenSolver's order), column norms / scaling / residual /
// gather streams.
#include <cooperative_groups.h>

#include <cstdlib>

#include "common.cuh"
#include "ritz_kernels.hpp"

namespace cg = cooperative_groups;

namespace fl {

// ------------------------------------------------------------------ streams
__global__ void symmetrize_kernel(const double* __restrict__ M, long ldm, int p, double* S,
                                  long lds) {
    const long total = (long)p * p;
    for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long)gridDim.x * blockDim.x) {
        const int j = (int)(e / p), i = (int)(e - (long)j * p);
        S[(long)j * lds + i] = 0.5 * (M[(long)j * ldm + i] + M[(long)i * ldm + j]);
    }
}
void launch_symmetrize(const double* M, long ldm, int p, double* S, long lds, cudaStream_t s) {
    if (p <= 0) return;
    symmetrize_kernel<<<148 * 2, 256, 0, s>>>(M, ldm, p, S, lds);
}

__global__ void set_diag_kernel(double* M, long ld, int from, int to, double v) {
    int i = from + blockIdx.x * blockDim.x + threadIdx.x;
    if (i < to) M[(long)i * ld + i] = v;
}
void launch_set_diag(double* M, long ld, int from, int to, double v, cudaStream_t s) {
    if (to <= from) return;
    set_diag_kernel<<<(to - from + 255) / 256, 256, 0, s>>>(M, ld, from, to, v);
}

// column 2-norms, fixed-shape tree reduction (run-to-run deterministic)
__global__ void col_norms_kernel(const double* __restrict__ X, long ldx, int n, double* norms) {
    const int c = blockIdx.x;
    const double* x = X + (long)c * ldx;
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += x[i] * x[i];
    s = warp_sum(s);
    __shared__ double red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];
        norms[c] = sqrt(t);
    }
}
void launch_col_norms(const double* X, long ldx, int n, int p, double* norms, cudaStream_t s) {
    if (p <= 0) return;
    col_norms_kernel<<<p, 256, 0, s>>>(X, ldx, n, norms);
}

// X[:, j] /= d[j]
__global__ void col_div_kernel(double* X, long ldx, int n, const double* __restrict__ d) {
    const int c = blockIdx.y;
    const double dv = d[c];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        X[(long)c * ldx + i] /= dv;
}
void launch_col_div(double* X, long ldx, int n, int p, const double* d, cudaStream_t s) {
    if (p <= 0) return;
    col_div_kernel<<<dim3((n + 255) / 256, p), 256, 0, s>>>(X, ldx, n, d);
}

// R = AV - V diag(lam)   (Eigen evaluates A*V into a temporary, then subtracts)
__global__ void residual_kernel(const double* __restrict__ AV, long ldav, const double* __restrict__ V,
                                long ldv, int n, const double* __restrict__ lam, double* R,
                                long ldr) {
    const int c = blockIdx.y;
    const double l = lam[c];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        R[(long)c * ldr + i] = AV[(long)c * ldav + i] - V[(long)c * ldv + i] * l;
}
void launch_residual(const double* AV, long ldav, const double* V, long ldv, int n, int p,
                     const double* lam, double* R, long ldr, cudaStream_t s) {
    if (p <= 0) return;
    residual_kernel<<<dim3((n + 255) / 256, p), 256, 0, s>>>(AV, ldav, V, ldv, n, lam, R, ldr);
}

// dst[:, j] = src[:, idx[j]] for j < k; columns k..kpad-1 of dst zeroed
__global__ void gather_cols_kernel(const double* __restrict__ src, long lds, int n,
                                   const int* __restrict__ idx, int k, double* dst, long ldd) {
    const int c = blockIdx.y;
    const double* s = c < k ? src + (long)idx[c] * lds : nullptr;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        dst[(long)c * ldd + i] = s ? s[i] : 0.0;
}
void launch_gather_cols(const double* src, long lds, int n, const int* idx, int k, int kpad,
                        double* dst, long ldd, cudaStream_t s) {
    if (kpad <= 0) return;
    gather_cols_kernel<<<dim3((n + 255) / 256, kpad), 256, 0, s>>>(src, lds, n, idx, k, dst, ldd);
}

// ------------------------------------------------------------------ Cholesky
// Diagonal 64x64 block, in shared memory, the reference's column algorithm
// (proj/src/ritz.cpp:64-79) on the already-updated block; reports the first
// pivot s <= 0 or non-finite (global index kb + j) into info[0..1].
struct CholInfo {
    int index;   // -1 = ok
    double pivot;
};

__global__ void __launch_bounds__(256) chol_diag_kernel(double* B, long ld, int kb, int limit,
                                                        CholInfo* info) {
    __shared__ double L[64][65];
    __shared__ int fail;
    const int tid = threadIdx.x;
    if (info->index >= 0) return;  // an earlier block already failed
    for (int e = tid; e < 64 * 64; e += 256) {
        const int i = e & 63, k = e >> 6;
        L[i][k] = B[(long)(kb + k) * ld + kb + i];
    }
    if (tid == 0) fail = 0;
    __syncthreads();
    for (int j = 0; j < 64; ++j) {
        if (tid == 0) {
            double s = L[j][j];
            for (int k = 0; k < j; ++k) s -= L[j][k] * L[j][k];
            if (kb + j < limit && (!(s > 0.0) || !isfinite(s))) {
                info->index = kb + j;
                info->pivot = s;
                fail = 1;
            }
            L[j][j] = sqrt(s);
        }
        __syncthreads();
        if (fail) return;
        for (int i = j + 1 + tid; i < 64; i += 256) {
            double t = L[i][j];
            for (int k = 0; k < j; ++k) t -= L[i][k] * L[j][k];
            L[i][j] = t / L[j][j];
        }
        __syncthreads();
    }
    for (int e = tid; e < 64 * 64; e += 256) {
        const int i = e & 63, k = e >> 6;
        B[(long)(kb + k) * ld + kb + i] = (i >= k) ? L[i][k] : 0.0;
    }
}

// rows i in [kb+64, P): L[i, kb:kb+64] = B[i, kb:kb+64] L_kk^{-T}
__global__ void __launch_bounds__(128) chol_panel_kernel(double* B, long ld, int kb, int P,
                                                         const CholInfo* info) {
    __shared__ double L[64][65];
    if (info->index >= 0) return;
    for (int e = threadIdx.x; e < 64 * 64; e += 128) {
        const int i = e & 63, k = e >> 6;
        L[i][k] = B[(long)(kb + k) * ld + kb + i];
    }
    __syncthreads();
    const int row = kb + 64 + blockIdx.x * 128 + threadIdx.x;
    if (row >= P) return;
    double x[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) {
        double t = B[(long)(kb + j) * ld + row];
#pragma unroll
        for (int k = 0; k < j; ++k) t -= x[k] * L[j][k];
        x[j] = t / L[j][j];
    }
#pragma unroll
    for (int j = 0; j < 64; ++j) B[(long)(kb + j) * ld + row] = x[j];
}

void launch_cholesky(double* B, long ld, int p, int P, void* info_dev, cudaStream_t s) {
    CholInfo* info = static_cast<CholInfo*>(info_dev);
    for (int kb = 0; kb < P; kb += 64) {
        chol_diag_kernel<<<1, 256, 0, s>>>(B, ld, kb, p, info);
        const int rest = P - kb - 64;
        if (rest > 0) {
            chol_panel_kernel<<<(rest + 127) / 128, 128, 0, s>>>(B, ld, kb, P, info);
            DGemm g{rest, rest, 64, B + (long)kb * ld + kb + 64, ld, 0,
                    B + (long)kb * ld + kb + 64, ld, 0,
                    B + (long)(kb + 64) * ld + kb + 64, ld, 0, -1.0, 1.0};
            launch_dgemm(g, false, true, 1, s);
        }
    }
}

// zero the strict upper triangle (L from the in-place Cholesky)
__global__ void tril_kernel(double* B, long ld, int P) {
    const long total = (long)P * P;
    for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long)gridDim.x * blockDim.x) {
        const int j = (int)(e / P), i = (int)(e - (long)j * P);
        if (i < j) B[(long)j * ld + i] = 0.0;
    }
}
void launch_tril(double* B, long ld, int P, cudaStream_t s) {
    tril_kernel<<<148, 256, 0, s>>>(B, ld, P);
}

// ------------------------------------------------------------------ real triangular 64x64 blocks
// X[r0:r0+64, :] <- T^{-1} X or T^{-T} X, T = L[k0:k0+64, k0:k0+64] lower non-unit.
template <bool TRANS>
__global__ void __launch_bounds__(128) dtrsm64_kernel(const double* L, long ldl, int k0, double* X,
                                                      long ldx, int r0, int ncols) {
    __shared__ double T[64][65];
    __shared__ double S[64][17];
    const int tid = threadIdx.x, c0 = blockIdx.x * 16;
    for (int e = tid; e < 64 * 64; e += 128) {
        const int i = e & 63, k = e >> 6;
        T[i][k] = L[(long)(k0 + k) * ldl + k0 + i];
    }
    for (int e = tid; e < 64 * 16; e += 128) {
        const int i = e & 63, c = e >> 6;
        S[i][c] = (c0 + c < ncols) ? X[(long)(c0 + c) * ldx + r0 + i] : 0.0;
    }
    __syncthreads();
    const int col = tid & 15, q = tid >> 4;
    if (!TRANS) {  // forward: T lower
        for (int r = 0; r < 64; ++r) {
            if (q == (r & 7)) S[r][col] /= T[r][r];
            __syncthreads();
            const double x = S[r][col];
            for (int i = q; i < 64; i += 8)
                if (i > r) S[i][col] -= T[i][r] * x;
            __syncthreads();
        }
    } else {  // backward with T^T (upper): (T^T)[i][r] = T[r][i]
        for (int r = 63; r >= 0; --r) {
            if (q == (r & 7)) S[r][col] /= T[r][r];
            __syncthreads();
            const double x = S[r][col];
            for (int i = q; i < r; i += 8) S[i][col] -= T[r][i] * x;
            __syncthreads();
        }
    }
    for (int e = tid; e < 64 * 16; e += 128) {
        const int i = e & 63, c = e >> 6;
        if (c0 + c < ncols) X[(long)(c0 + c) * ldx + r0 + i] = S[i][c];
    }
}

// X <- L^{-1} X (trans=false) or L^{-T} X (trans=true); L P x P lower with
// identity padding, X P x ncols (ncols multiple of 64).
void launch_trsm_lower(const double* L, long ldl, int P, double* X, long ldx, int ncols, bool trans,
                       cudaStream_t s) {
    const int NB = P / 64;
    const int grid = (ncols + 15) / 16;
    if (!trans) {
        for (int ib = 0; ib < NB; ++ib) {
            dtrsm64_kernel<false><<<grid, 128, 0, s>>>(L, ldl, ib * 64, X, ldx, ib * 64, ncols);
            const int rest = P - (ib + 1) * 64;
            if (rest > 0) {
                DGemm g{rest, ncols, 64, L + (long)(ib * 64) * ldl + (ib + 1) * 64, ldl, 0,
                        X + ib * 64, ldx, 0, X + (ib + 1) * 64, ldx, 0, -1.0, 1.0};
                launch_dgemm(g, false, false, 1, s);
            }
        }
    } else {
        for (int ib = NB - 1; ib >= 0; --ib) {
            dtrsm64_kernel<true><<<grid, 128, 0, s>>>(L, ldl, ib * 64, X, ldx, ib * 64, ncols);
            const int above = ib * 64;
            if (above > 0) {
                // X[0:above] -= (L[ib*64:+64, 0:above])^T X[ib*64:+64]
                DGemm g{above, ncols, 64, L + ib * 64, ldl, 0, X + ib * 64, ldx, 0, X, ldx, 0,
                        -1.0, 1.0};
                launch_dgemm(g, true, false, 1, s);
            }
        }
    }
}

// ------------------------------------------------------------------ Jacobi eigensolver
// Parallel cyclic two-sided Jacobi with the round-robin (circle) ordering:
// round r pairs (r, pe-1) and ((r+k) mod (pe-1), (r-k) mod (pe-1)), k >= 1.
// Every CTA recomputes all rotations of the round from the current matrix
// (double-buffered, so no intra-round hazards), then applies its share of the
// 2x2 block updates A' = J^T A J and V' = V J: one grid barrier per round.
// Rotations follow Golub & Van Loan sym.schur2; a pair is skipped when
// |a_ab| <= thr = eps * ||A||_F. Converged when a sweep rotates nothing.
struct JacobiArgs {
    double* A0;
    double* A1;
    long lda;
    double* V;
    long ldv;
    int p;       // true size
    int pe;      // even size (p or p+1)
    double thr;  // skip threshold
    int max_sweeps;
    int* sweeps_done;
    unsigned long long* rot_count;  // per sweep counter, [max_sweeps]
};

__device__ __forceinline__ void round_pair(int r, int k, int pe, int& a, int& b) {
    const int m = pe - 1;
    if (k == 0) {
        a = r;
        b = m;
    } else {
        a = (r + k) % m;
        b = (r - k + m) % m;
    }
    if (a > b) {
        int t = a;
        a = b;
        b = t;
    }
}

__global__ void __launch_bounds__(256) jacobi_kernel(JacobiArgs J) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double jsh[];
    const int half = J.pe / 2;
    double* cs = jsh;              // [half]
    double* sn = jsh + half;       // [half]
    double* tt = jsh + 2 * half;   // [half] (t for the diagonal update)
    int* pa = reinterpret_cast<int*>(jsh + 3 * half);  // [half]
    int* pb = pa + half;                               // [half]
    int* role = pb + half;                             // [pe]: pair index * 2 + (is_b)
    __shared__ unsigned long long cnt;
    const int p = J.p, pe = J.pe;
    const long lda = J.lda;
    double* Acur = J.A0;
    double* Anext = J.A1;
    auto el = [&](const double* M, int i, int j) -> double {
        if (i >= p || j >= p) return 0.0;
        return M[(long)j * lda + i];
    };
    int sweep = 0;
    const long gthreads = (long)gridDim.x * blockDim.x;
    const long gtid = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long nblk = (long)half * (half + 1) / 2;
    const long nv = (long)p * half;
    // each phase below issues all of a thread's loads before using any of them,
    // so a round costs one L2 round trip per phase plus the grid barrier
    constexpr int BATCH = 4;
    for (; sweep < J.max_sweeps; ++sweep) {
        for (int r = 0; r < pe - 1; ++r) {
            if (threadIdx.x == 0) cnt = 0;
            __syncthreads();
            // rotations of this round (every CTA, redundantly; half <= 4 * 256)
            unsigned long long local = 0;
            {
                int ka[BATCH], kb_[BATCH];
                double apq[BATCH], app[BATCH], aqq[BATCH];
#pragma unroll
                for (int u = 0; u < BATCH; ++u) {
                    const int k = threadIdx.x + u * blockDim.x;
                    ka[u] = -1;
                    kb_[u] = -1;
                    if (k < half) {
                        round_pair(r, k, pe, ka[u], kb_[u]);
                        const bool ok = kb_[u] < p;
                        apq[u] = ok ? Acur[(long)kb_[u] * lda + ka[u]] : 0.0;
                        app[u] = ok ? Acur[(long)ka[u] * lda + ka[u]] : 0.0;
                        aqq[u] = ok ? Acur[(long)kb_[u] * lda + kb_[u]] : 0.0;
                    }
                }
#pragma unroll
                for (int u = 0; u < BATCH; ++u) {
                    const int k = threadIdx.x + u * blockDim.x;
                    if (k >= half) continue;
                    pa[k] = ka[u];
                    pb[k] = kb_[u];
                    double c = 1.0, sn_ = 0.0, t = 0.0;
                    if (kb_[u] < p && fabs(apq[u]) > J.thr) {
                        const double tau = (aqq[u] - app[u]) / (2.0 * apq[u]);
                        t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        c = 1.0 / sqrt(1.0 + t * t);
                        sn_ = t * c;
                        ++local;
                    }
                    cs[k] = c;
                    sn[k] = sn_;
                    tt[k] = t;
                }
            }
            if (local) atomicAdd(&cnt, local);
            __syncthreads();
            if (blockIdx.x == 0 && threadIdx.x == 0 && cnt) atomicAdd(&J.rot_count[sweep], cnt);
            // apply: 2x2 blocks (P, Q), P <= Q only (A' symmetric: also written
            // transposed); V' = V J on column pairs
            for (long e0 = gtid; e0 < nblk; e0 += BATCH * gthreads) {
                double B[BATCH][4];
                int PQ[BATCH][2];
#pragma unroll
                for (int u = 0; u < BATCH; ++u) {
                    const long e = e0 + u * gthreads;
                    PQ[u][0] = -1;
                    if (e >= nblk) continue;
                    int Q = (int)((sqrt(8.0 * (double)e + 1.0) - 1.0) * 0.5);
                    while ((long)Q * (Q + 1) / 2 > e) --Q;
                    while ((long)(Q + 1) * (Q + 2) / 2 <= e) ++Q;
                    const int P = (int)(e - (long)Q * (Q + 1) / 2);
                    PQ[u][0] = P;
                    PQ[u][1] = Q;
                    B[u][0] = el(Acur, pa[P], pa[Q]);
                    B[u][1] = el(Acur, pa[P], pb[Q]);
                    B[u][2] = el(Acur, pb[P], pa[Q]);
                    B[u][3] = el(Acur, pb[P], pb[Q]);
                }
#pragma unroll
                for (int u = 0; u < BATCH; ++u) {
                    const int P = PQ[u][0], Q = PQ[u][1];
                    if (P < 0) continue;
                    const int a1 = pa[P], b1 = pb[P], a2 = pa[Q], b2 = pb[Q];
                    const double c1 = cs[P], s1 = sn[P], c2 = cs[Q], s2 = sn[Q];
                    const double Baa = B[u][0], Bab = B[u][1], Bba = B[u][2], Bbb = B[u][3];
                    double naa, nab, nba, nbb;
                    if (P == Q && s1 != 0.0) {
                        const double t = tt[P];
                        naa = Baa - t * Bab;
                        nbb = Bbb + t * Bab;
                        nab = 0.0;
                        nba = 0.0;
                    } else {
                        // rows: x_a = c1*row_a - s1*row_b ; x_b = s1*row_a + c1*row_b
                        const double ra_a = c1 * Baa - s1 * Bba, ra_b = c1 * Bab - s1 * Bbb;
                        const double rb_a = s1 * Baa + c1 * Bba, rb_b = s1 * Bab + c1 * Bbb;
                        naa = ra_a * c2 - ra_b * s2;
                        nab = ra_a * s2 + ra_b * c2;
                        nba = rb_a * c2 - rb_b * s2;
                        nbb = rb_a * s2 + rb_b * c2;
                    }
                    if (a1 < p && a2 < p) Anext[(long)a2 * lda + a1] = naa;
                    if (a1 < p && b2 < p) Anext[(long)b2 * lda + a1] = nab;
                    if (b1 < p && a2 < p) Anext[(long)a2 * lda + b1] = nba;
                    if (b1 < p && b2 < p) Anext[(long)b2 * lda + b1] = nbb;
                    if (P != Q) {
                        if (a1 < p && a2 < p) Anext[(long)a1 * lda + a2] = naa;
                        if (a1 < p && b2 < p) Anext[(long)a1 * lda + b2] = nab;
                        if (b1 < p && a2 < p) Anext[(long)b1 * lda + a2] = nba;
                        if (b1 < p && b2 < p) Anext[(long)b1 * lda + b2] = nbb;
                    }
                }
            }
            for (long e0 = gtid; e0 < nv; e0 += BATCH * gthreads) {
                double va[BATCH], vb[BATCH];
                int xs[BATCH], Ps[BATCH];
#pragma unroll
                for (int u = 0; u < BATCH; ++u) {
                    const long e = e0 + u * gthreads;
                    Ps[u] = -1;
                    if (e >= nv) continue;
                    const int x = (int)(e % p), P = (int)(e / p);
                    if (sn[P] == 0.0 || pb[P] >= p) continue;
                    Ps[u] = P;
                    xs[u] = x;
                    va[u] = J.V[(long)pa[P] * J.ldv + x];
                    vb[u] = J.V[(long)pb[P] * J.ldv + x];
                }
#pragma unroll
                for (int u = 0; u < BATCH; ++u) {
                    const int P = Ps[u];
                    if (P < 0) continue;
                    const double c1 = cs[P], s1 = sn[P];
                    J.V[(long)pa[P] * J.ldv + xs[u]] = c1 * va[u] - s1 * vb[u];
                    J.V[(long)pb[P] * J.ldv + xs[u]] = s1 * va[u] + c1 * vb[u];
                }
            }
            grid.sync();
            double* t = Acur;
            Acur = Anext;
            Anext = t;
        }
        // all CTAs see the same counter after the last barrier of the sweep
        const unsigned long long total = *(volatile unsigned long long*)&J.rot_count[sweep];
        if (total == 0) {
            ++sweep;
            break;
        }
    }
    // leave the final matrix in A0
    if (Acur != J.A0) {
        const long total = (long)p * p;
        for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
             e += (long)gridDim.x * blockDim.x) {
            const int j = (int)(e / p), i = (int)(e - (long)j * p);
            J.A0[(long)j * lda + i] = Acur[(long)j * lda + i];
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *J.sweeps_done = sweep;
}

// ascending sort of the diagonal with its eigenvector columns:
// rank(i) = #{j : d_j < d_i or (d_j == d_i and j < i)}
__global__ void eig_sort_kernel(const double* __restrict__ A, long lda, int p,
                                const double* __restrict__ V, long ldv, double* vals,
                                double* Vout, long ldo) {
    const int i = blockIdx.x;
    const double di = A[(long)i * lda + i];
    __shared__ int rank_s;
    int cnt = 0;
    for (int j = threadIdx.x; j < p; j += blockDim.x) {
        const double dj = A[(long)j * lda + j];
        cnt += (dj < di || (dj == di && j < i)) ? 1 : 0;
    }
    for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
    __shared__ int red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        rank_s = t;
        vals[t] = di;
    }
    __syncthreads();
    const int r = rank_s;
    for (int x = threadIdx.x; x < p; x += blockDim.x) Vout[(long)r * ldo + x] = V[(long)i * ldv + x];
}

__global__ void eye_kernel(double* V, long ldv, int rows, int cols) {
    const long total = (long)rows * cols;
    for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long)gridDim.x * blockDim.x) {
        const int j = (int)(e / rows), i = (int)(e - (long)j * rows);
        V[(long)j * ldv + i] = (i == j) ? 1.0 : 0.0;
    }
}

__global__ void fro2_kernel(const double* A, long lda, int p, double* out) {
    double s = 0.0;
    const long total = (long)p * p;
    for (long e = threadIdx.x; e < total; e += blockDim.x) {
        const int j = (int)(e / p), i = (int)(e - (long)j * p);
        const double v = A[(long)j * lda + i];
        s += v * v;
    }
    s = warp_sum(s);
    __shared__ double red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        *out = t;
    }
}

void launch_fro2(const double* A, long lda, int p, double* out_dev, cudaStream_t s) {
    fro2_kernel<<<1, 1024, 0, s>>>(A, lda, p, out_dev);
}

int jacobi_eig(double* A, long lda, int p, double fro, double* work, double* V, long ldv,
               double* vals, double* Vout, long ldo, int* scratch_int, unsigned long long* counters,
               int max_sweeps, cudaStream_t s) {
    if (p <= 0) return 0;
    const int pe = p + (p & 1);
    const int half = pe / 2;
    eye_kernel<<<148, 256, 0, s>>>(V, ldv, p, p);
    cudaMemsetAsync(counters, 0, sizeof(unsigned long long) * max_sweeps, s);
    JacobiArgs J;
    J.A0 = A;
    J.A1 = work;
    J.lda = lda;
    J.V = V;
    J.ldv = ldv;
    J.p = p;
    J.pe = pe;
    J.thr = 2.220446049250313e-16 * fro;
    if (!(J.thr > 0.0)) J.thr = 0.0;
    J.max_sweeps = max_sweeps;
    J.sweeps_done = scratch_int;
    J.rot_count = counters;
    const size_t sm = sizeof(double) * 3 * half + sizeof(int) * (2 * half + pe);
    ensure_smem((const void*)jacobi_kernel, sm);
    int dev = 0, nsm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_kernel, 256, sm);
    if (per_sm < 1) per_sm = 1;
    int blocks = nsm * (per_sm > 2 ? 2 : per_sm);
    const long work_items = (long)half * half;
    if (work_items < (long)blocks * 256) {
        blocks = (int)((work_items + 255) / 256);
        if (blocks < 1) blocks = 1;
    }
    if (const char* e = getenv("FL_JACOBI_BLOCKS")) {
        const int want = atoi(e);
        if (want > 0 && want < blocks) blocks = want;
    }
    void* args[] = {&J};
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)jacobi_kernel, dim3(blocks), dim3(256),
                                                args, sm, s);
    if (e != cudaSuccess) return -1;
    eig_sort_kernel<<<p, 256, 0, s>>>(A, lda, p, V, ldv, vals, Vout, ldo);
    return 0;
}

// ------------------------------------------------------------------ block Jacobi
// Two-sided block Jacobi (cyclic round-robin over 32-wide column blocks):
// per outer round, each of the P/64 disjoint block pairs (a, b) is solved in
// one CTA by cyclic scalar Jacobi in shared memory (same sym.schur2
// rotations and skip threshold eps ||A||_F as above), giving a 64 x 64
// orthogonal Q_ab; then one launch applies all of them: A[I, J] <- Q_I^T
// A[I, J] Q_J for every pair-tile (I, J) and V[:, J] <- V[:, J] Q_J. An outer
// sweep visits every block pair once, so a sweep that rotates nothing leaves
// every |a_pq| <= thr: the scalar kernel's stopping rule. Grid-wide
// synchronisation drops from p - 1 barriers per sweep to 2 (P/32 - 1).
constexpr int BJ = 32;       // column block
constexpr int BJ2 = 2 * BJ;  // pair subproblem
constexpr int BJL = BJ2 + 1; // padded smem leading dimension

__device__ __forceinline__ int bj_global(int l, int ia, int ib) {
    return l < BJ ? ia * BJ + l : ib * BJ + (l - BJ);
}

__global__ void __launch_bounds__(256) bj_inner_kernel(const double* __restrict__ W, long ld, int nb,
                                                       int r, double thr, int max_inner,
                                                       double* __restrict__ Qbuf,
                                                       unsigned long long* cnt) {
    extern __shared__ double bsm[];
    double* S = bsm;              // [BJ2][BJL], column-major
    double* Q = bsm + BJ2 * BJL;  // [BJ2][BJL]
    __shared__ double rc[BJ], rs[BJ], rt[BJ];
    __shared__ int pa[BJ], pb[BJ];
    __shared__ int any;
    const int tid = threadIdx.x;
    int ia, ib;
    round_pair(r, blockIdx.x, nb, ia, ib);
    for (int e = tid; e < BJ2 * BJ2; e += blockDim.x) {
        const int lr = e % BJ2, lc = e / BJ2;
        S[lc * BJL + lr] = W[(long)bj_global(lc, ia, ib) * ld + bj_global(lr, ia, ib)];
        Q[lc * BJL + lr] = (lr == lc) ? 1.0 : 0.0;
    }
    __syncthreads();
    unsigned long long rot = 0;
    for (int sw = 0; sw < max_inner; ++sw) {
        if (tid == 0) any = 0;
        __syncthreads();
        for (int rr = 0; rr < BJ2 - 1; ++rr) {
            if (tid < BJ) {
                int a, b;
                round_pair(rr, tid, BJ2, a, b);
                const double apq = S[b * BJL + a], app = S[a * BJL + a], aqq = S[b * BJL + b];
                double c = 1.0, sn_ = 0.0, t = 0.0;
                if (fabs(apq) > thr) {
                    const double tau = (aqq - app) / (2.0 * apq);
                    t = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                    c = 1.0 / sqrt(1.0 + t * t);
                    sn_ = t * c;
                    ++rot;
                    any = 1;
                }
                pa[tid] = a;
                pb[tid] = b;
                rc[tid] = c;
                rs[tid] = sn_;
                rt[tid] = t;
            }
            __syncthreads();
            // S <- J^T S J on 2 x 2 blocks (P rows, Q cols), in place
            for (int e = tid; e < BJ * BJ; e += blockDim.x) {
                const int P = e % BJ, Qc = e / BJ;
                const double s1 = rs[P], s2 = rs[Qc];
                if (s1 == 0.0 && s2 == 0.0) continue;
                const int a1 = pa[P], b1 = pb[P], a2 = pa[Qc], b2 = pb[Qc];
                const double c1 = rc[P], c2 = rc[Qc];
                const double Baa = S[a2 * BJL + a1], Bab = S[b2 * BJL + a1];
                const double Bba = S[a2 * BJL + b1], Bbb = S[b2 * BJL + b1];
                double naa, nab, nba, nbb;
                if (P == Qc) {
                    const double t = rt[P];
                    naa = Baa - t * Bab;
                    nbb = Bbb + t * Bab;
                    nab = 0.0;
                    nba = 0.0;
                } else {
                    const double ra_a = c1 * Baa - s1 * Bba, ra_b = c1 * Bab - s1 * Bbb;
                    const double rb_a = s1 * Baa + c1 * Bba, rb_b = s1 * Bab + c1 * Bbb;
                    naa = ra_a * c2 - ra_b * s2;
                    nab = ra_a * s2 + ra_b * c2;
                    nba = rb_a * c2 - rb_b * s2;
                    nbb = rb_a * s2 + rb_b * c2;
                }
                S[a2 * BJL + a1] = naa;
                S[b2 * BJL + a1] = nab;
                S[a2 * BJL + b1] = nba;
                S[b2 * BJL + b1] = nbb;
            }
            // Q <- Q J
            for (int e = tid; e < BJ2 * BJ; e += blockDim.x) {
                const int x = e % BJ2, P = e / BJ2;
                const double sn_ = rs[P];
                if (sn_ == 0.0) continue;
                const double c = rc[P];
                const double qa = Q[pa[P] * BJL + x], qb = Q[pb[P] * BJL + x];
                Q[pa[P] * BJL + x] = c * qa - sn_ * qb;
                Q[pb[P] * BJL + x] = sn_ * qa + c * qb;
            }
            __syncthreads();
        }
        if (!any) break;
        __syncthreads();
    }
    double* Qo = Qbuf + (long)blockIdx.x * BJ2 * BJ2;
    for (int e = tid; e < BJ2 * BJ2; e += blockDim.x) {
        const int lr = e % BJ2, lc = e / BJ2;
        Qo[lc * BJ2 + lr] = Q[lc * BJL + lr];
    }
    if (tid < BJ) {
        for (int off = 16; off > 0; off >>= 1) rot += __shfl_xor_sync(0xffffffffu, rot, off);
        if (tid == 0 && rot) atomicAdd(cnt, rot);
    }
}

// C (64 x 64, smem ld BJL) = op(X) Y with X, Y 64 x 64 in smem (ld BJL);
// TX: X transposed. 256 threads, 4 x 4 outputs each.
template <bool TX>
__device__ __forceinline__ void bj_mm(const double* X, const double* Y, double* C) {
    const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int k = 0; k < BJ2; ++k) {
        double xv[4], yv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int row = ty + 16 * i;
            xv[i] = TX ? X[row * BJL + k] : X[k * BJL + row];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) yv[j] = Y[(tx + 16 * j) * BJL + k];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fma(xv[i], yv[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) C[(tx + 16 * j) * BJL + ty + 16 * i] = acc[i][j];
}

// CTA t < ntA: A pair-tile (I, J), I <= J (symmetric: the transposed tile is
// written too); otherwise a 64-row tile of V times Q_J.
__global__ void __launch_bounds__(256) bj_update_kernel(double* __restrict__ W, long ld,
                                                        double* __restrict__ V, long ldv, int P,
                                                        int nb, int r,
                                                        const double* __restrict__ Qbuf) {
    extern __shared__ double usm[];
    double* X = usm;
    double* QI = usm + BJ2 * BJL;
    double* QJ = usm + 2 * BJ2 * BJL;
    double* T = usm + 3 * BJ2 * BJL;
    const int np = nb / 2;
    const int ntA = np * (np + 1) / 2;
    const int tid = threadIdx.x;
    auto loadQ = [&](int k, double* dst) {
        const double* q = Qbuf + (long)k * BJ2 * BJ2;
        for (int e = tid; e < BJ2 * BJ2; e += blockDim.x) dst[(e / BJ2) * BJL + e % BJ2] = q[e];
    };
    if ((int)blockIdx.x < ntA) {
        int t = blockIdx.x, I = 0;
        while (t >= np - I) {
            t -= np - I;
            ++I;
        }
        const int J = I + t;
        int ia, ib, ja, jb;
        round_pair(r, I, nb, ia, ib);
        round_pair(r, J, nb, ja, jb);
        for (int e = tid; e < BJ2 * BJ2; e += blockDim.x) {
            const int lr = e % BJ2, lc = e / BJ2;
            X[lc * BJL + lr] = W[(long)bj_global(lc, ja, jb) * ld + bj_global(lr, ia, ib)];
        }
        loadQ(I, QI);
        loadQ(J, QJ);
        __syncthreads();
        bj_mm<false>(X, QJ, T);  // T = X Q_J
        __syncthreads();
        bj_mm<true>(QI, T, X);   // X = Q_I^T T
        __syncthreads();
        for (int e = tid; e < BJ2 * BJ2; e += blockDim.x) {
            const int lr = e % BJ2, lc = e / BJ2;
            const double v = X[lc * BJL + lr];
            W[(long)bj_global(lc, ja, jb) * ld + bj_global(lr, ia, ib)] = v;
        }
        if (I != J)
            for (int e = tid; e < BJ2 * BJ2; e += blockDim.x) {
                const int lr = e % BJ2, lc = e / BJ2;  // element (lr of J-set, lc of I-set)
                W[(long)bj_global(lc, ia, ib) * ld + bj_global(lr, ja, jb)] = X[lr * BJL + lc];
            }
    } else {
        const int v = blockIdx.x - ntA;
        const int rt = v % (P / BJ2), J = v / (P / BJ2);
        int ja, jb;
        round_pair(r, J, nb, ja, jb);
        const int r0 = rt * BJ2;
        for (int e = tid; e < BJ2 * BJ2; e += blockDim.x) {
            const int lr = e % BJ2, lc = e / BJ2;
            X[lc * BJL + lr] = V[(long)bj_global(lc, ja, jb) * ldv + r0 + lr];
        }
        loadQ(J, QJ);
        __syncthreads();
        bj_mm<false>(X, QJ, T);
        __syncthreads();
        for (int e = tid; e < BJ2 * BJ2; e += blockDim.x) {
            const int lr = e % BJ2, lc = e / BJ2;
            V[(long)bj_global(lc, ja, jb) * ldv + r0 + lr] = T[lc * BJL + lr];
        }
    }
}

__global__ void bj_prepare_kernel(const double* __restrict__ A, long lda, int p, int P,
                                  double* __restrict__ W, double* __restrict__ V) {
    const long total = (long)P * P;
    for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long)gridDim.x * blockDim.x) {
        const int j = (int)(e / P), i = (int)(e - (long)j * P);
        W[e] = (i < p && j < p) ? A[(long)j * lda + i] : 0.0;
        V[e] = (i == j) ? 1.0 : 0.0;
    }
}

int block_jacobi_eig(const double* A, long lda, int p, int P, double fro, double* W, double* V,
                     double* Qbuf, double* vals, double* Vout, long ldo,
                     unsigned long long* counters, unsigned long long* h_counter, int max_sweeps,
                     int* sweeps_out, cudaStream_t s) {
    if (p <= 0) return 0;
    if (P % BJ2 != 0 || P < p) return -1;
    const int nb = P / BJ;
    const int np = nb / 2;
    const double thr = fro > 0.0 ? 2.220446049250313e-16 * fro : 0.0;
    bj_prepare_kernel<<<148, 256, 0, s>>>(A, lda, p, P, W, V);
    const size_t sm_in = sizeof(double) * 2 * BJ2 * BJL;
    const size_t sm_up = sizeof(double) * 4 * BJ2 * BJL;
    ensure_smem((const void*)bj_inner_kernel, sm_in);
    ensure_smem((const void*)bj_update_kernel, sm_up);
    const int ntiles = np * (np + 1) / 2 + (P / BJ2) * np;
    // a single pair (P = 64) is the whole problem: iterate it to convergence
    const int max_inner = np == 1 ? max_sweeps : 1;
    cudaMemsetAsync(counters, 0, sizeof(unsigned long long) * max_sweeps, s);
    int sweep = 0;
    for (; sweep < max_sweeps; ++sweep) {
        for (int r = 0; r < nb - 1; ++r) {
            bj_inner_kernel<<<np, 256, sm_in, s>>>(W, P, nb, r, thr, max_inner, Qbuf,
                                                   counters + sweep);
            bj_update_kernel<<<ntiles, 256, sm_up, s>>>(W, P, V, P, P, nb, r, Qbuf);
        }
        cudaMemcpyAsync(h_counter, counters + sweep, sizeof(unsigned long long),
                        cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) return -1;
        if (*h_counter == 0) {
            ++sweep;
            break;
        }
    }
    if (sweeps_out) *sweeps_out = sweep;
    eig_sort_kernel<<<p, 256, 0, s>>>(W, P, p, V, P, vals, Vout, ldo);
    return 0;
}

}  // namespace fl

namespace fl {

// ------------------------------------------------------------------ column-pivoted Householder QR
// ColPivHouseholderQR stand-in (proj/src/ritz.cpp:22-29, drivers.cpp:33-36),
// LAPACK dgeqp3/dlaqp2 semantics: pivot = largest remaining partial column
// norm (first on ties), Householder beta = -sign(alpha) ||x||, partial norms
// downdated with the sqrt(eps) recompute guard. One cooperative kernel: per
// step, CTA 0 picks the pivot, swaps and forms the reflector; every CTA then
// applies it to its share of the trailing columns (2 grid barriers / step).
struct QRArgs {
    double* A;
    long lda;
    int n, p, kmax;
    double* tau;   // [kmax]
    int* jpvt;     // [p]
    double* vn1;   // [p] partial norms
    double* vn2;   // [p] reference norms
};

__device__ double block_sum(double v, double* red) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    return t;
}

__global__ void __launch_bounds__(256) qr_kernel(QRArgs q) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double red[32];
    __shared__ int s_piv;
    __shared__ double s_beta, s_scale;
    const long lda = q.lda;
    // initial norms
    for (int j = blockIdx.x; j < q.p; j += gridDim.x) {
        double s = 0.0;
        for (int i = threadIdx.x; i < q.n; i += blockDim.x) s += q.A[(long)j * lda + i] * q.A[(long)j * lda + i];
        s = block_sum(s, red);
        if (threadIdx.x == 0) {
            q.vn1[j] = sqrt(s);
            q.vn2[j] = sqrt(s);
            q.jpvt[j] = j;
        }
    }
    grid.sync();
    const double tol3z = sqrt(2.220446049250313e-16);
    for (int k = 0; k < q.kmax; ++k) {
        if (blockIdx.x == 0) {
            if (threadIdx.x == 0) {
                int pv = k;
                double best = q.vn1[k];
                for (int j = k + 1; j < q.p; ++j)
                    if (q.vn1[j] > best) { best = q.vn1[j]; pv = j; }
                s_piv = pv;
                if (pv != k) {
                    const int t = q.jpvt[k];
                    q.jpvt[k] = q.jpvt[pv];
                    q.jpvt[pv] = t;
                    q.vn1[pv] = q.vn1[k];
                    q.vn2[pv] = q.vn2[k];
                }
            }
            __syncthreads();
            const int pv = s_piv;
            double* ck = q.A + (long)k * lda;
            if (pv != k) {
                double* cp = q.A + (long)pv * lda;
                for (int i = threadIdx.x; i < q.n; i += blockDim.x) {
                    const double t = ck[i];
                    ck[i] = cp[i];
                    cp[i] = t;
                }
            }
            __syncthreads();
            // reflector for column k (dlarfg)
            double s = 0.0;
            for (int i = k + 1 + threadIdx.x; i < q.n; i += blockDim.x) s += ck[i] * ck[i];
            const double xnorm = sqrt(block_sum(s, red));
            if (threadIdx.x == 0) {
                const double alpha = ck[k];
                if (xnorm == 0.0) {
                    q.tau[k] = 0.0;
                    s_beta = alpha;
                    s_scale = 1.0;
                } else {
                    const double beta = -copysign(hypot(alpha, xnorm), alpha);
                    q.tau[k] = (beta - alpha) / beta;
                    s_beta = beta;
                    s_scale = 1.0 / (alpha - beta);
                }
            }
            __syncthreads();
            if (q.tau[k] != 0.0)
                for (int i = k + 1 + threadIdx.x; i < q.n; i += blockDim.x) ck[i] *= s_scale;
            __syncthreads();
            if (threadIdx.x == 0) ck[k] = s_beta;
        }
        grid.sync();
        // apply H_k = I - tau v v^T (v_k = 1) to columns k+1.. and downdate norms
        const double tk = q.tau[k];
        const double* v = q.A + (long)k * lda;
        for (int j = k + 1 + blockIdx.x; j < q.p; j += gridDim.x) {
            double* cj = q.A + (long)j * lda;
            if (tk != 0.0) {
                double s = (threadIdx.x == 0) ? cj[k] : 0.0;
                for (int i = k + 1 + threadIdx.x; i < q.n; i += blockDim.x) s += v[i] * cj[i];
                const double w = tk * block_sum(s, red);
                if (threadIdx.x == 0) cj[k] -= w;
                for (int i = k + 1 + threadIdx.x; i < q.n; i += blockDim.x) cj[i] -= w * v[i];
                __syncthreads();
            }
            const double v1 = q.vn1[j], v2 = q.vn2[j], rkj = cj[k];
            __syncthreads();
            if (v1 != 0.0) {  // dlaqp2 norm downdate
                double temp = fabs(rkj) / v1;
                temp = fmax(0.0, 1.0 - temp * temp);
                const double r = v1 / v2;
                const double temp2 = temp * r * r;
                if (temp2 <= tol3z) {
                    double s = 0.0;
                    for (int i = k + 1 + threadIdx.x; i < q.n; i += blockDim.x) s += cj[i] * cj[i];
                    const double nr = sqrt(block_sum(s, red));
                    if (threadIdx.x == 0) {
                        q.vn1[j] = nr;
                        q.vn2[j] = nr;
                    }
                } else if (threadIdx.x == 0) {
                    q.vn1[j] = v1 * sqrt(temp);
                }
            }
            __syncthreads();
        }
        grid.sync();
    }
}

// Q[:, 0:r] = H_0 ... H_{r-1} I[:, 0:r] (dorg2r), reflectors in A below the diagonal
struct OrgArgs {
    const double* A;
    long lda;
    const double* tau;
    double* Q;
    long ldq;
    int n, r;
};

__global__ void __launch_bounds__(256) orgqr_kernel(OrgArgs o) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double red[32];
    for (int j = blockIdx.x; j < o.r; j += gridDim.x)
        for (int i = threadIdx.x; i < o.n; i += blockDim.x)
            o.Q[(long)j * o.ldq + i] = (i == j) ? 1.0 : 0.0;
    grid.sync();
    for (int k = o.r - 1; k >= 0; --k) {
        const double tk = o.tau[k];
        const double* v = o.A + (long)k * o.lda;
        if (tk != 0.0)
            for (int j = k + blockIdx.x; j < o.r; j += gridDim.x) {
                double* qj = o.Q + (long)j * o.ldq;
                double s = (threadIdx.x == 0) ? qj[k] : 0.0;
                for (int i = k + 1 + threadIdx.x; i < o.n; i += blockDim.x) s += v[i] * qj[i];
                const double w = tk * block_sum(s, red);
                if (threadIdx.x == 0) qj[k] -= w;
                for (int i = k + 1 + threadIdx.x; i < o.n; i += blockDim.x) qj[i] -= w * v[i];
                __syncthreads();
            }
        grid.sync();
    }
}

static int coop_blocks(const void* fn, int work) {
    int dev = 0, nsm = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0);
    int blocks = nsm * (per_sm > 0 ? 1 : 1);
    if (work < blocks) blocks = work > 0 ? work : 1;
    return blocks;
}

int launch_qr(double* A, long lda, int n, int p, double* tau, int* jpvt, double* vn1, double* vn2,
              cudaStream_t s) {
    QRArgs q{A, lda, n, p, n < p ? n : p, tau, jpvt, vn1, vn2};
    void* args[] = {&q};
    const int blocks = coop_blocks((const void*)qr_kernel, p);
    return cudaLaunchCooperativeKernel((const void*)qr_kernel, dim3(blocks), dim3(256), args, 0, s) ==
                   cudaSuccess
               ? 0
               : -1;
}

int launch_orgqr(const double* A, long lda, const double* tau, int n, int r, double* Q, long ldq,
                 cudaStream_t s) {
    if (r <= 0) return 0;
    OrgArgs o{A, lda, tau, Q, ldq, n, r};
    void* args[] = {&o};
    const int blocks = coop_blocks((const void*)orgqr_kernel, r);
    return cudaLaunchCooperativeKernel((const void*)orgqr_kernel, dim3(blocks), dim3(256), args, 0,
                                       s) == cudaSuccess
               ? 0
               : -1;
}

}  // namespace fl
