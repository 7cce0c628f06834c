// Complex partial-pivot LU of z I - A and the blocked multi-RHS solve
// (NodeFactorization, proj/src/filterop.cpp:9-32), batched over contour nodes.
//
//  shift        F = z I - A                          HBM stream, (8 + 16 G) N^2 B / G nodes
//  panel        64-wide panel, partial pivoting      panel.cu (8-CTA cluster,
//                                                    register-resident leaves)
//  laswp        row interchanges outside the panel   one gather/scatter per panel
//  trinv        64x64 diagonal-block inverses        triangular solves become GEMMs
//  zgemm        trailing update / solve updates      DMMA (gemm.cu)
#include <cooperative_groups.h>
#include <cstdlib>
#include <cstring>

#include <mutex>
#include <map>
#include <utility>

#include "common.cuh"
#include "kernels.hpp"

namespace cg = cooperative_groups;

namespace fl {

void ensure_smem(const void* func, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    size_t& have = done[{func, dev}];
    if (bytes > have) {
        launch_check(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes),
                     "cudaFuncSetAttribute(max dynamic shared memory)");
        have = bytes;
    }
}

void ensure_attr(const void* func, cudaFuncAttribute attr, int value) {
    static std::mutex mu;
    static std::map<std::pair<std::pair<const void*, int>, int>, int> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(std::make_pair(func, dev), (int)attr);
    auto it = done.find(key);
    if (it != done.end() && it->second == value) return;
    launch_check(cudaFuncSetAttribute(func, attr, value), "cudaFuncSetAttribute");
    done[key] = value;
}

// ------------------------------------------------------------------ shift
// One thread per row pair of a column: A's pair is read once (16-byte load)
// and written, negated and shifted, into every node of the batch (16-byte
// stores per plane), so a launch moves 8 N^2 + 16 N^2 G bytes. Rows are the
// fast grid axis (blockIdx.x), columns blockIdx.y: no 64-bit index division.
__global__ void __launch_bounds__(256) shift_kernel(const double* __restrict__ A, long lda, int N,
                                                    ZBatch F, NodeShifts z, int batch) {
    const int c = blockIdx.y;
    const int r = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (r >= N) return;
    const double2 a = __ldcs(reinterpret_cast<const double2*>(A + (long)c * lda + r));
    const long o = (long)c * F.ld + r;
    const int d = c - r;  // 0 or 1: the diagonal element of this pair, if any
    for (int b = 0; b < batch; ++b) {
        double2 re = make_double2(-a.x, -a.y), im = make_double2(0.0, 0.0);
        if (d == 0) {
            re.x += z.zr[b];
            im.x = z.zi[b];
        } else if (d == 1) {
            re.y += z.zr[b];
            im.y = z.zi[b];
        }
        *reinterpret_cast<double2*>(F.re + b * F.stride + o) = re;
        *reinterpret_cast<double2*>(F.im + b * F.stride + o) = im;
    }
}

void launch_shift(const double* A, long lda, int N, ZBatch F, const NodeShifts& z, int batch,
                  cudaStream_t s) {
    if (N <= 0 || batch <= 0) return;
    // N is a multiple of the 64-wide tile; lda, F.ld even and A 16-byte aligned
    shift_kernel<<<dim3((N / 2 + 255) / 256, N), 256, 0, s>>>(A, lda, N, F, z, batch);
}

// ------------------------------------------------------------------ panel
// panel.cu: register-resident two-level cluster panel (launch_panel).
constexpr int PW = 64;

// ------------------------------------------------------------------ laswp
// The panel's 64 interchanges applied to the columns outside the panel as one
// gather/scatter of the <= 128 moved rows (net permutation from the panel
// kernel): every load of a CTA is issued before any store.
constexpr int LS_COLS = 16;
__global__ void __launch_bounds__(256) laswp_panel_kernel(ZBatch F, int a0, int a1, int b0,
                                                          int b1, const int* __restrict__ ptab) {
    __shared__ double vr[2 * PW][LS_COLS + 1];
    __shared__ double vi[2 * PW][LS_COLS + 1];
    __shared__ int pos[2 * PW], src[2 * PW];
    const int b = blockIdx.y;
    const int* tab = ptab + (long)b * (4 * PW + 1);
    const int cnt = tab[0];
    for (int m = threadIdx.x; m < cnt; m += blockDim.x) {
        pos[m] = tab[1 + m];
        src[m] = tab[1 + 2 * PW + m];
    }
    __syncthreads();
    const int na = a1 - a0, ncols = na + (b1 - b0);
    double* Fr = F.re + b * F.stride;
    double* Fi = F.im + b * F.stride;
    const int c0 = blockIdx.x * LS_COLS;
    for (int e = threadIdx.x; e < cnt * LS_COLS; e += blockDim.x) {
        const int m = e % cnt, c = e / cnt;
        const int k = c0 + c;
        if (k >= ncols) continue;
        const int col = k < na ? a0 + k : b0 + (k - na);
        const long o = (long)col * F.ld + src[m];
        vr[m][c] = Fr[o];
        vi[m][c] = Fi[o];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < cnt * LS_COLS; e += blockDim.x) {
        const int m = e % cnt, c = e / cnt;
        const int k = c0 + c;
        if (k >= ncols) continue;
        const int col = k < na ? a0 + k : b0 + (k - na);
        const long o = (long)col * F.ld + pos[m];
        Fr[o] = vr[m][c];
        Fi[o] = vi[m][c];
    }
}

// Warp-per-column form: lane l moves entries l, l+32, l+64, l+96 of the net
// permutation for WC columns, every load of the warp issued (8 WC in flight
// per lane, no shared-memory round trip) before its stores; columns are
// independent, so a __syncwarp orders the gather before the scatter.
constexpr int LW_WC = 2;  // columns per warp
__global__ void __launch_bounds__(256) laswp_warp_kernel(ZBatch F, int a0, int a1, int b0, int b1,
                                                         const int* __restrict__ ptab) {
    const int b = blockIdx.y, lane = threadIdx.x & 31;
    const int* tab = ptab + (long)b * (4 * PW + 1);
    const int cnt = __ldg(tab);
    int pos[4], src[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int m = lane + 32 * q;
        pos[q] = m < cnt ? __ldg(tab + 1 + m) : 0;
        src[q] = m < cnt ? __ldg(tab + 1 + 2 * PW + m) : 0;
    }
    const int na = a1 - a0, ncols = na + (b1 - b0);
    const int k0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * LW_WC;
    double* Fr = F.re + b * F.stride;
    double* Fi = F.im + b * F.stride;
    long cb[LW_WC];
#pragma unroll
    for (int w = 0; w < LW_WC; ++w) {
        const int k = k0 + w;
        cb[w] = k < ncols ? (long)(k < na ? a0 + k : b0 + (k - na)) * F.ld : -1;
    }
    double vr[LW_WC][4], vi[LW_WC][4];
#pragma unroll
    for (int w = 0; w < LW_WC; ++w)
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (cb[w] >= 0 && lane + 32 * q < cnt) {
                vr[w][q] = Fr[cb[w] + src[q]];
                vi[w][q] = Fi[cb[w] + src[q]];
            }
    __syncwarp();
#pragma unroll
    for (int w = 0; w < LW_WC; ++w)
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (cb[w] >= 0 && lane + 32 * q < cnt) {
                Fr[cb[w] + pos[q]] = vr[w][q];
                Fi[cb[w] + pos[q]] = vi[w][q];
            }
}

void launch_laswp(ZBatch F, int a0, int a1, int b0, int b1, const int* ptab, int batch,
                  cudaStream_t s) {
    a1 = a1 > a0 ? a1 : a0;
    b1 = b1 > b0 ? b1 : b0;
    const int ncols = (a1 - a0) + (b1 - b0);
    if (ncols <= 0) return;
    static const bool smem_form = [] {
        const char* e = std::getenv("FEASTLAB_LASWP");
        return e && std::strcmp(e, "smem") == 0;
    }();
    if (smem_form) {
        laswp_panel_kernel<<<dim3((ncols + LS_COLS - 1) / LS_COLS, batch), 256, 0, s>>>(
            F, a0, a1, b0, b1, ptab);
        return;
    }
    constexpr int per_cta = 8 * LW_WC;
    laswp_warp_kernel<<<dim3((ncols + per_cta - 1) / per_cta, batch), 256, 0, s>>>(F, a0, a1, b0,
                                                                                  b1, ptab);
}

// ------------------------------------------------------------------ outer-block laswp
// The np panels of an outer block leave np net permutations; the columns
// outside the block need only their composition, applied in ONE pass: the
// block's own bw = 64 np rows are then written as whole lines (no sector fill
// for a partial write), and each displaced row below the block is read and
// written once instead of once per panel that touched it.
//
// compose_perm_kernel: cmap[r] = the row whose data sits at position r (identity
// on entry and on exit); a panel table moves cmap[src] to pos. Table written
// per node: [0] count of moved rows below the block, then the source row of
// each of the block's rows, then (position, source) of the moved rows below.
__global__ void __launch_bounds__(128) compose_perm_kernel(const int* __restrict__ ptab,
                                                           long panel_stride, int np, int k0,
                                                           int N, int* cmap_all, int* btab_all) {
    const int b = blockIdx.x, t = threadIdx.x;
    int* cmap = cmap_all + (long)b * N;
    int* out = btab_all + (long)b * LB_TAB;
    __shared__ int rc;
    if (t == 0) rc = 0;
    for (int j = 0; j < np; ++j) {
        const int* tab = ptab + j * panel_stride + (long)b * (4 * PW + 1);
        const int cnt = tab[0];
        int v = 0;
        if (t < cnt) v = cmap[tab[1 + 2 * PW + t]];
        __syncthreads();
        if (t < cnt) cmap[tab[1 + t]] = v;
        __syncthreads();
    }
    const int bw = np * PW, c0 = k0 + bw;
    for (int i = t; i < bw; i += blockDim.x) {
        out[1 + i] = cmap[k0 + i];
        cmap[k0 + i] = k0 + i;
    }
    for (int j = 0; j < np; ++j) {
        const int* tab = ptab + j * panel_stride + (long)b * (4 * PW + 1);
        const int cnt = tab[0];
        if (t < cnt) {
            const int p = tab[1 + t];
            if (p >= c0) {
                const int v = atomicExch(&cmap[p], p);  // first claim lists it, and resets
                if (v != p) {
                    const int s = atomicAdd(&rc, 1);
                    out[1 + LB_MAX + s] = p;
                    out[1 + 2 * LB_MAX + s] = v;
                }
            }
        }
    }
    __syncthreads();
    if (t == 0) out[0] = rc;
}

__global__ void iota_kernel(int* a, long n, int period) {
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = (int)(i % period);
}

// LB_CW columns per CTA; thread t owns block rows t + 256 q and moved rows
// t + 256 q below the block. Every load of the CTA is issued before the barrier,
// every store after it (a column's sources and positions overlap).
constexpr int LB_CW = 2, LB_Q = LB_MAX / 256;
__global__ void __launch_bounds__(256) laswp_block_kernel(ZBatch F, int k0, int bw, int a0,
                                                          int a1, int b0, int b1,
                                                          const int* __restrict__ btab) {
    const int b = blockIdx.y, t = threadIdx.x;
    const int* tab = btab + (long)b * LB_TAB;
    const int rc = __ldg(tab);
    int ds[LB_Q], rp[LB_Q], rs[LB_Q];
#pragma unroll
    for (int q = 0; q < LB_Q; ++q) {
        const int i = t + 256 * q;
        ds[q] = i < bw ? __ldg(tab + 1 + i) : -1;
        if (ds[q] == k0 + i) ds[q] = -1;  // stays
        rp[q] = i < rc ? __ldg(tab + 1 + LB_MAX + i) : -1;
        rs[q] = i < rc ? __ldg(tab + 1 + 2 * LB_MAX + i) : -1;
    }
    const int na = a1 - a0, ncols = na + (b1 - b0);
    double* Fr = F.re + b * F.stride;
    double* Fi = F.im + b * F.stride;
    long cb[LB_CW];
#pragma unroll
    for (int w = 0; w < LB_CW; ++w) {
        const int k = blockIdx.x * LB_CW + w;
        cb[w] = k < ncols ? (long)(k < na ? a0 + k : b0 + (k - na)) * F.ld : -1;
    }
    double dr[LB_CW][LB_Q], di[LB_CW][LB_Q], vr[LB_CW][LB_Q], vi[LB_CW][LB_Q];
#pragma unroll
    for (int w = 0; w < LB_CW; ++w)
#pragma unroll
        for (int q = 0; q < LB_Q; ++q) {
            if (cb[w] >= 0 && ds[q] >= 0) {
                dr[w][q] = Fr[cb[w] + ds[q]];
                di[w][q] = Fi[cb[w] + ds[q]];
            }
            if (cb[w] >= 0 && rs[q] >= 0) {
                vr[w][q] = Fr[cb[w] + rs[q]];
                vi[w][q] = Fi[cb[w] + rs[q]];
            }
        }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < LB_CW; ++w)
#pragma unroll
        for (int q = 0; q < LB_Q; ++q) {
            if (cb[w] >= 0 && ds[q] >= 0) {
                Fr[cb[w] + k0 + t + 256 * q] = dr[w][q];
                Fi[cb[w] + k0 + t + 256 * q] = di[w][q];
            }
            if (cb[w] >= 0 && rs[q] >= 0) {
                Fr[cb[w] + rp[q]] = vr[w][q];
                Fi[cb[w] + rp[q]] = vi[w][q];
            }
        }
}

void launch_perm_identity(int* cmap, int N, int batch, cudaStream_t s) {
    const long n = (long)N * batch;
    iota_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(cmap, n, N);
}

void launch_laswp_block(ZBatch F, int N, int k0, int np, int a0, int a1, int b0, int b1,
                        const int* ptab, long panel_stride, int* cmap, int* btab, int batch,
                        cudaStream_t s) {
    a1 = a1 > a0 ? a1 : a0;
    b1 = b1 > b0 ? b1 : b0;
    const int ncols = (a1 - a0) + (b1 - b0);
    if (ncols <= 0 || np <= 0) return;
    compose_perm_kernel<<<batch, 128, 0, s>>>(ptab, panel_stride, np, k0, N, cmap, btab);
    laswp_block_kernel<<<dim3((ncols + LB_CW - 1) / LB_CW, batch), 256, 0, s>>>(
        F, k0, np * PW, a0, a1, b0, b1, btab);
}

// ------------------------------------------------------------------ 64x64 triangular inverses
// Inverse of the unit-lower (L) or upper (U) 64x64 diagonal block at (r0, r0)
// of every node, by substitution on the identity in shared memory. The
// triangular solves then become DMMA GEMMs (zgemm SET) with these blocks.
// 256 threads: thread (col = tid & 63, q = tid >> 6) owns rows q, q+4, ...
struct InvShared {
    double Tr[PW][PW + 1];
    double Ti[PW][PW + 1];
    double Xr[PW][PW + 1];
    double Xi[PW][PW + 1];
};

template <bool UPPER>
__global__ void __launch_bounds__(256) trinv_kernel(ZBatch T, int r0, int blk_stride_nodes,
                                                    ZBatch Inv, int first_block) {
    extern __shared__ __align__(16) unsigned char raw[];
    InvShared& sh = *reinterpret_cast<InvShared*>(raw);
    const int b = blockIdx.y;
    const int blk = first_block + blockIdx.x;
    const int k0 = r0 + blockIdx.x * PW;
    const double* Tr = T.re + b * T.stride;
    const double* Ti = T.im + b * T.stride;
    const int tid = threadIdx.x;
    for (int e = tid; e < PW * PW; e += 256) {
        const int i = e & (PW - 1), k = e >> 6;
        const long o = (long)(k0 + k) * T.ld + k0 + i;
        sh.Tr[i][k] = Tr[o];
        sh.Ti[i][k] = Ti[o];
        sh.Xr[i][k] = (i == k) ? 1.0 : 0.0;
        sh.Xi[i][k] = 0.0;
    }
    __syncthreads();
    const int col = tid & 63, q = tid >> 6;
    if (!UPPER) {
        for (int r = 0; r < PW - 1; ++r) {
            const cplx x{sh.Xr[r][col], sh.Xi[r][col]};
            for (int i = q; i < PW; i += 4) {
                if (i > r) {
                    const cplx l{sh.Tr[i][r], sh.Ti[i][r]};
                    sh.Xr[i][col] -= l.re * x.re - l.im * x.im;
                    sh.Xi[i][col] -= l.re * x.im + l.im * x.re;
                }
            }
            __syncthreads();
        }
    } else {
        for (int r = PW - 1; r >= 0; --r) {
            if (q == (r & 3)) {
                const cplx inv = crecip(cplx{sh.Tr[r][r], sh.Ti[r][r]});
                const cplx y = cmul(cplx{sh.Xr[r][col], sh.Xi[r][col]}, inv);
                sh.Xr[r][col] = y.re;
                sh.Xi[r][col] = y.im;
            }
            __syncthreads();
            const cplx x{sh.Xr[r][col], sh.Xi[r][col]};
            for (int i = q; i < r; i += 4) {
                const cplx u{sh.Tr[i][r], sh.Ti[i][r]};
                sh.Xr[i][col] -= u.re * x.re - u.im * x.im;
                sh.Xi[i][col] -= u.re * x.im + u.im * x.re;
            }
            __syncthreads();
        }
    }
    double* Ir = Inv.re + b * Inv.stride + (long)blk * PW * PW;
    double* Ii = Inv.im + b * Inv.stride + (long)blk * PW * PW;
    for (int e = tid; e < PW * PW; e += 256) {
        const int i = e & (PW - 1), k = e >> 6;
        Ir[(long)k * PW + i] = sh.Xr[i][k];
        Ii[(long)k * PW + i] = sh.Xi[i][k];
    }
    (void)blk_stride_nodes;
}

void launch_trinv(ZBatch T, int r0, int nblocks, bool upper, ZBatch Inv, int first_block,
                  int batch, cudaStream_t s) {
    if (nblocks <= 0) return;
    const size_t sm = sizeof(InvShared);
    if (upper) {
        ensure_smem((const void*)trinv_kernel<true>, sm);
        trinv_kernel<true><<<dim3(nblocks, batch), 256, sm, s>>>(T, r0, 0, Inv, first_block);
    } else {
        ensure_smem((const void*)trinv_kernel<false>, sm);
        trinv_kernel<false><<<dim3(nblocks, batch), 256, sm, s>>>(T, r0, 0, Inv, first_block);
    }
}

// ------------------------------------------------------------------ pivots -> permutation
__global__ void ipiv_to_perm_kernel(const int* __restrict__ ipiv, int* __restrict__ perm, int N) {
    const int b = blockIdx.x;
    const int* ip = ipiv + (long)b * N;
    int* pm = perm + (long)b * N;
    if (threadIdx.x == 0) {
        for (int i = 0; i < N; ++i) pm[i] = i;
        for (int i = 0; i < N; ++i) {
            const int p = ip[i];
            if (p != i) {
                int t = pm[i];
                pm[i] = pm[p];
                pm[p] = t;
            }
        }
    }
}

void launch_ipiv_to_perm(const int* ipiv, int* perm, int N, int batch, cudaStream_t s) {
    ipiv_to_perm_kernel<<<batch, 32, 0, s>>>(ipiv, perm, N);
}

__global__ void permute_rhs_kernel(const double* __restrict__ X, long ldx, int N, int P,
                                   const int* __restrict__ perm, ZBatch W) {
    const int b = blockIdx.z;
    const int c = blockIdx.y;
    const int* pm = perm + (long)b * N;
    double* Wr = W.re + b * W.stride + (long)c * W.ld;
    double* Wi = W.im + b * W.stride + (long)c * W.ld;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
        Wr[i] = X[(long)c * ldx + pm[i]];
        Wi[i] = 0.0;
    }
}

void launch_permute_rhs(const double* X, long ldx, int N, int P, const int* perm, ZBatch W,
                        int batch, cudaStream_t s) {
    if (P <= 0) return;
    permute_rhs_kernel<<<dim3((N + 255) / 256, P, batch), 256, 0, s>>>(X, ldx, N, P, perm, W);
}

// ------------------------------------------------------------------ ordered accumulation
// Y = [Y +] sum_b Re(w_b W_b), b ascending; Re(w W) = wr*Wr - wi*Wi with the
// two products and the difference each rounded (std::complex product, no FMA),
// exactly as proj/src/filterop.cpp:80 evaluates it.
__global__ void accumulate_kernel(ZBatch W, int N, int P, NodeShifts w, int batch, double* Y,
                                  long ldy, bool add) {
    const int c = blockIdx.y;
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= N) return;
    double y = add ? Y[(long)c * ldy + r] : 0.0;
    const long oc = (long)c * W.ld + r;
    for (int b = 0; b < batch; ++b) {
        const long o = b * W.stride + oc;
        const double t = __dsub_rn(__dmul_rn(w.zr[b], __ldcs(W.re + o)),
                                   __dmul_rn(w.zi[b], __ldcs(W.im + o)));
        y = __dadd_rn(y, t);
    }
    Y[(long)c * ldy + r] = y;
}

void launch_accumulate(ZBatch W, int N, int P, const NodeShifts& w, int batch, double* Y, long ldy,
                       bool add_to_Y, cudaStream_t s) {
    if (P <= 0 || N <= 0) return;
    accumulate_kernel<<<dim3((N + 255) / 256, P), 256, 0, s>>>(W, N, P, w, batch, Y, ldy, add_to_Y);
}

// G-invariant reduction (fl_ctx_set_reduction ORDERED): every rank writes its
// nodes' terms t_b = Re(w_b W_b) (the same two rounded products and rounded
// difference as accumulate_kernel); after an all-gather every rank sums all
// n_c terms in ascending global node order, which is accumulate_kernel's
// association on one GPU: Y is bitwise the same at every GPU count.
__global__ void node_terms_kernel(ZBatch W, int N, int P, NodeShifts w, int batch, double* T,
                                  long tstride) {
    const long total = (long)N * P;
    const int b = blockIdx.y;
    for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long)gridDim.x * blockDim.x) {
        const long c = e / N, r = e - c * N;
        const long o = b * W.stride + c * W.ld + r;
        T[b * tstride + e] = __dsub_rn(__dmul_rn(w.zr[b], W.re[o]), __dmul_rn(w.zi[b], W.im[o]));
    }
}

__global__ void ordered_sum_kernel(const double* __restrict__ T, long tstride, NodeSlots sl, int nc,
                                   int N, int P, double* Y, long ldy, bool add) {
    const long total = (long)N * P;
    for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long)gridDim.x * blockDim.x) {
        const long c = e / N, r = e - c * N;
        double y = add ? Y[c * ldy + r] : 0.0;
        for (int k = 0; k < nc; ++k) y = __dadd_rn(y, T[sl.slot[k] * tstride + e]);
        Y[c * ldy + r] = y;
    }
}

void launch_node_terms(ZBatch W, int N, int P, const NodeShifts& w, int batch, double* T,
                       long tstride, cudaStream_t s) {
    if (P <= 0 || batch <= 0) return;
    node_terms_kernel<<<dim3(148 * 4 / batch + 1, batch), 256, 0, s>>>(W, N, P, w, batch, T,
                                                                       tstride);
}

void launch_ordered_sum(const double* T, long tstride, const NodeSlots& sl, int nc, int N, int P,
                        double* Y, long ldy, bool add_to_Y, cudaStream_t s) {
    if (P <= 0) return;
    ordered_sum_kernel<<<148 * 4, 256, 0, s>>>(T, tstride, sl, nc, N, P, Y, ldy, add_to_Y);
}

// ------------------------------------------------------------------ singularity check
__global__ void check_diag_kernel(ZBatch F, int n, int offset, int* bad_node) {
    const int b = blockIdx.y;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const long o = b * F.stride + (long)i * F.ld + i;
        const double d = hypot(F.re[o], F.im[o]);
        if (!(d > 0.0) || !isfinite(d)) atomicMin(bad_node, offset + b);
    }
}

void launch_check_diag(ZBatch F, int n, int batch, int offset, int* bad_node, cudaStream_t s) {
    check_diag_kernel<<<dim3((n + 255) / 256, batch), 256, 0, s>>>(F, n, offset, bad_node);
}

}  // namespace fl
