// Device-side fixture generation: the seeded orthogonal
// factor and the dense test matrix of proj/src/matmodel.cpp:93-119 --
// Householder QR of the seeded Gaussian block, Q = H_1 ... H_n I, columns
// sign-normalised so their largest-magnitude entry is positive, and
// A = Q diag(lambda) Q^T, symmetrised.
//
// Blocked Householder QR (dgeqrf / dorgqr with compact-WY block reflectors,
// nb = 64): the panel is factored by a cooperative level-2 kernel (one CTA per
// panel column, grid barriers between column steps); the block reflector
// I - V T V^T is applied to the trailing matrix, and to Q on the way back,
// by three DMMA GEMMs (dgemm_kernel). Everything works on the padded order
// N = round_up(n, 64): the padding block of G is the identity, whose
// reflectors are H = I (tau = 0), so Q's padding block is the identity too.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.hpp"
#include "ritz_kernels.hpp"

namespace cg = cooperative_groups;

namespace fl {

namespace {

constexpr int NB = 64;

__device__ double fx_block_sum(double v, double* red) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    return t;
}

// Unpivoted Householder QR of the panel A[k0:N, k0:k0+NB] (dgeqr2): reflector j
// has v_j = 1 implied, the rest of v stored below the diagonal, R on and above.
__global__ void __launch_bounds__(256) hqr_panel_kernel(double* A, long lda, int N, int k0,
                                                        double* tau) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double red[32];
    __shared__ double s_beta, s_scale;
    for (int j = 0; j < NB; ++j) {
        const int k = k0 + j;
        double* ck = A + (long)k * lda;
        if (blockIdx.x == 0) {  // dlarfg on column k
            double s = 0.0;
            for (int i = k + 1 + threadIdx.x; i < N; i += blockDim.x) s += ck[i] * ck[i];
            const double xnorm = sqrt(fx_block_sum(s, red));
            if (threadIdx.x == 0) {
                const double alpha = ck[k];
                if (xnorm == 0.0) {
                    tau[k] = 0.0;
                    s_beta = alpha;
                    s_scale = 1.0;
                } else {
                    const double beta = -copysign(hypot(alpha, xnorm), alpha);
                    tau[k] = (beta - alpha) / beta;
                    s_beta = beta;
                    s_scale = 1.0 / (alpha - beta);
                }
            }
            __syncthreads();
            if (tau[k] != 0.0)
                for (int i = k + 1 + threadIdx.x; i < N; i += blockDim.x) ck[i] *= s_scale;
            __syncthreads();
            if (threadIdx.x == 0) ck[k] = s_beta;
        }
        grid.sync();
        const double tk = tau[k];
        if (tk != 0.0)  // H_k on the panel's remaining columns
            for (int c = k + 1 + blockIdx.x; c < k0 + NB; c += gridDim.x) {
                double* cj = A + (long)c * lda;
                double s = (threadIdx.x == 0) ? cj[k] : 0.0;
                for (int i = k + 1 + threadIdx.x; i < N; i += blockDim.x) s += ck[i] * cj[i];
                const double w = tk * fx_block_sum(s, red);
                if (threadIdx.x == 0) cj[k] -= w;
                for (int i = k + 1 + threadIdx.x; i < N; i += blockDim.x) cj[i] -= w * ck[i];
                __syncthreads();
            }
        grid.sync();
    }
}

// V (N x NB, ld N): the panel's reflectors as an explicit unit lower trapezoid
// (zero above row k0 + j in column j, one on it).
__global__ void __launch_bounds__(256) hqr_copy_v_kernel(const double* A, long lda, int N, int k0,
                                                         double* V) {
    const int j = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int d = k0 + j;
    V[(long)j * N + i] = i < d ? 0.0 : (i == d ? 1.0 : A[(long)d * lda + i]);
}

// T (NB x NB upper triangular, dlarft forward / columnwise) from G = V^T V:
// T[j][j] = tau_j, T[0:j, j] = -tau_j T[0:j, 0:j] G[0:j, j]. One CTA.
__global__ void __launch_bounds__(64) hqr_t_kernel(const double* G, const double* tau, double* T) {
    __shared__ double t[NB][NB + 1];
    const int i = threadIdx.x;
    for (int j = 0; j < NB; ++j) t[i][j] = 0.0;
    __syncthreads();
    for (int j = 0; j < NB; ++j) {
        const double tj = tau[j];
        double s = 0.0;
        if (i < j)
            for (int l = i; l < j; ++l) s += t[i][l] * G[(long)j * NB + l];
        __syncthreads();
        if (i < j) t[i][j] = -tj * s;
        if (i == j) t[i][j] = tj;
        __syncthreads();
    }
    for (int j = 0; j < NB; ++j) T[(long)j * NB + i] = t[i][j];
}

__global__ void __launch_bounds__(256) fx_identity_kernel(double* Q, long ld, int N) {
    const int j = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N) Q[(long)j * ld + i] = i == j ? 1.0 : 0.0;
}

// proj/src/matmodel.cpp:101-105: a column whose largest-magnitude entry (first
// one on ties, Eigen's maxCoeff) is negative is negated. One CTA per column.
__global__ void __launch_bounds__(256) fx_sign_kernel(double* Q, long ld, int n) {
    __shared__ double sv[256];
    __shared__ int si[256];
    double* q = Q + (long)blockIdx.x * ld;
    double best = -1.0;
    int idx = 0x7fffffff;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double a = fabs(q[i]);
        if (a > best) {
            best = a;
            idx = i;
        }
    }
    sv[threadIdx.x] = best;
    si[threadIdx.x] = idx;
    __syncthreads();
    for (int off = 128; off > 0; off >>= 1) {
        if (threadIdx.x < off) {
            const double b = sv[threadIdx.x + off];
            const int bi = si[threadIdx.x + off];
            if (b > sv[threadIdx.x] || (b == sv[threadIdx.x] && bi < si[threadIdx.x])) {
                sv[threadIdx.x] = b;
                si[threadIdx.x] = bi;
            }
        }
        __syncthreads();
    }
    const bool flip = q[si[0]] < 0.0;
    __syncthreads();
    if (flip)
        for (int i = threadIdx.x; i < n; i += blockDim.x) q[i] = -q[i];
}

// B[:, j] = Q[:, j] * vals[j] (j < n; padding columns zero)
__global__ void __launch_bounds__(256) fx_scale_cols_kernel(const double* Q, long ld, int N, int n,
                                                            const double* vals, double* B) {
    const int j = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N) B[(long)j * ld + i] = j < n ? Q[(long)j * ld + i] * vals[j] : 0.0;
}

}  // namespace

// In-place blocked Householder QR of the N x N matrix A (ld N; N multiple of
// 64), then Q (N x N, ld N) = H_1 ... H_N I. Work: V (N x 64), W (64 x N), W2
// (64 x N), G (64 x 64), T (N/64 x 64 x 64), tau (N). Returns 0 on success.
int fixture_householder_q(double* A, int N, double* Q, double* V, double* W, double* W2, double* G,
                          double* T, double* tau, cudaStream_t s) {
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = nsm < NB ? nsm : NB;
    const dim3 g1((N + 255) / 256, NB);
    for (int k0 = 0; k0 < N; k0 += NB) {
        const long lda = N;
        int kk = k0;
        int NN = N;
        void* args[] = {&A, (void*)&lda, &NN, &kk, &tau};
        if (cudaLaunchCooperativeKernel((const void*)hqr_panel_kernel, dim3(blocks), dim3(256), args,
                                        0, s) != cudaSuccess)
            return -1;
        hqr_copy_v_kernel<<<g1, 256, 0, s>>>(A, N, N, k0, V);
        // rows < k0 of V are zero: every product below runs over rows k0..N
        const int R = N - k0;
        const double* Vk = V + k0;
        DGemm gg{NB, NB, R, Vk, N, 0, Vk, N, 0, G, NB, 0, 1.0, 0.0};  // G = V^T V
        launch_dgemm(gg, true, false, 1, s);
        double* Tk = T + (long)(k0 / NB) * NB * NB;
        hqr_t_kernel<<<1, NB, 0, s>>>(G, tau + k0, Tk);
        const int m = N - k0 - NB;  // trailing columns
        if (m > 0) {
            double* At = A + (long)(k0 + NB) * N + k0;
            // W = V^T A_trail;  W2 = T^T W;  A_trail -= V W2   (H_nb ... H_1 = I - V T^T V^T)
            DGemm g1_{NB, m, R, Vk, N, 0, At, N, 0, W, NB, 0, 1.0, 0.0};
            launch_dgemm(g1_, true, false, 1, s);
            DGemm g2_{NB, m, NB, Tk, NB, 0, W, NB, 0, W2, NB, 0, 1.0, 0.0};
            launch_dgemm(g2_, true, false, 1, s);
            DGemm g3_{R, m, NB, Vk, N, 0, W2, NB, 0, At, N, 0, -1.0, 1.0};
            launch_dgemm(g3_, false, false, 1, s);
        }
    }
    // Q = H_1 ... H_N I, block reflectors applied last to first (dorgqr)
    fx_identity_kernel<<<dim3((N + 255) / 256, N), 256, 0, s>>>(Q, N, N);
    for (int k0 = N - NB; k0 >= 0; k0 -= NB) {
        hqr_copy_v_kernel<<<g1, 256, 0, s>>>(A, N, N, k0, V);
        const double* Tk = T + (long)(k0 / NB) * NB * NB;
        // only rows and columns >= k0 of Q differ from the identity so far
        const int m = N - k0;
        double* Qs = Q + (long)k0 * N + k0;
        const double* Vk = V + k0;
        DGemm g1_{NB, m, m, Vk, N, 0, Qs, N, 0, W, NB, 0, 1.0, 0.0};
        launch_dgemm(g1_, true, false, 1, s);
        DGemm g2_{NB, m, NB, Tk, NB, 0, W, NB, 0, W2, NB, 0, 1.0, 0.0};
        launch_dgemm(g2_, false, false, 1, s);
        DGemm g3_{m, m, NB, Vk, N, 0, W2, NB, 0, Qs, N, 0, -1.0, 1.0};
        launch_dgemm(g3_, false, false, 1, s);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

void fixture_sign_normalize(double* Q, long ld, int n, cudaStream_t s) {
    if (n > 0) fx_sign_kernel<<<n, 256, 0, s>>>(Q, ld, n);
}

// A = 0.5 (M + M^T), M = Q diag(vals) Q^T (proj/src/matmodel.cpp:112-118). Q, A,
// B, M: N x N, ld N (B, M scratch); vals: n values on the device.
void fixture_assemble(const double* Q, const double* vals, int N, int n, double* B, double* M,
                      double* A, cudaStream_t s) {
    fx_scale_cols_kernel<<<dim3((N + 255) / 256, N), 256, 0, s>>>(Q, N, N, n, vals, B);
    DGemm g{N, N, N, B, N, 0, Q, N, 0, M, N, 0, 1.0, 0.0};
    launch_dgemm(g, false, true, 1, s);
    launch_symmetrize(M, N, N, A, N, s);
}

}  // namespace fl
