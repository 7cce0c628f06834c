// Complex partial-pivot LU of z I - A and the blocked multi-RHS solve
// (NodeFactorization, proj/src/filterop.cpp:9-32), batched over contour nodes.
//
//  shift        F = z I - A                          HBM stream, 24 N^2 B / node
//  panel        64-wide panel, partial pivoting      8-CTA cluster, DSMEM pivot
//                                                    exchange, 1 cluster barrier / column
//  laswp        row interchanges outside the panel
//  trsm         64x64 triangular blocks (unit-lower / upper) on a column strip
//  zgemm_sub    trailing update / solve updates      DMMA (gemm.cu)
#include <cooperative_groups.h>

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
        cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        have = bytes;
    }
}

// ------------------------------------------------------------------ shift
__global__ void shift_kernel(const double* __restrict__ A, long lda, int N, ZBatch F,
                             NodeShifts z) {
    const int b = blockIdx.y;
    double* Fr = F.re + b * F.stride;
    double* Fi = F.im + b * F.stride;
    const long total = (long)N * N;
    for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long)gridDim.x * blockDim.x) {
        const long c = e / N, r = e - c * N;
        double a = -A[c * lda + r];
        double im = 0.0;
        if (r == c) {
            a += z.zr[b];
            im = z.zi[b];
        }
        Fr[c * F.ld + r] = a;
        Fi[c * F.ld + r] = im;
    }
}

void launch_shift(const double* A, long lda, int N, ZBatch F, const NodeShifts& z, int batch,
                  cudaStream_t s) {
    int blocks = 148 * 4 / (batch > 0 ? batch : 1);
    if (blocks < 8) blocks = 8;
    shift_kernel<<<dim3(blocks, batch), 256, 0, s>>>(A, lda, N, F, z);
}

// ------------------------------------------------------------------ panel
// Cluster of PCL CTAs per node. CTA r owns panel rows [k0 + r*R, k0 + (r+1)*R).
// Per column j (one cluster barrier):
//   every CTA published (score, row) of its best candidate for column j plus a
//   copy of that candidate row's 64 panel entries, and the owner of row j a
//   copy of row j (double-buffered by j parity) -> after the barrier each CTA
//   reduces the PCL candidates (ties -> lowest row, Eigen's maxCoeff), takes the
//   pivot row from the winner's shared memory (DSMEM) and the owners of rows j
//   and piv write the interchanged rows; then each CTA scales its rows of
//   column j and applies the rank-1 update to the panel columns right of j,
//   fusing the candidate search for column j+1.
constexpr int PCL = 8;
constexpr int PTH = 512;
constexpr int PW = 64;

struct PanelShared {
    double cand_score[2];
    int cand_row[2];
    double cand_vals[2][2][PW];  // [parity][re/im][col]
    double diag_vals[2][2][PW];
    double u[2][PW];             // pivot row (this column)
    double red_s[PTH / 32];
    int red_i[PTH / 32];
    int piv;
    int winner;
    int pivs[PW];       // this panel's pivot rows (rank 0)
    int tpos[2 * PW];   // net row permutation of the panel: row tpos[m] <- row tsrc[m]
    int tsrc[2 * PW];
};

__global__ void __cluster_dims__(PCL, 1, 1) __launch_bounds__(PTH)
    panel_kernel(ZBatch F, int N, int k0, int* __restrict__ ipiv, int* __restrict__ ptab) {
    cg::cluster_group cluster = cg::this_cluster();
    __shared__ PanelShared sh;
    const int rank = (int)cluster.block_rank();
    const int b = blockIdx.y;
    double* Fr = F.re + b * F.stride;
    double* Fi = F.im + b * F.stride;
    const long ld = F.ld;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int rows_total = N - k0;
    const int R = (rows_total + PCL - 1) / PCL;
    const int lo = k0 + rank * R;
    const int hi = min(N, lo + R);

    auto at = [&](int r, int c) { return (long)c * ld + r; };

    // candidate search for column c over own rows >= rmin, then publish
    auto publish = [&](int c, int par, double s, int idx) {
        warp_argmax(s, idx);
        if (lane == 0) { sh.red_s[wid] = s; sh.red_i[wid] = idx; }
        __syncthreads();
        if (wid == 0) {
            double s2 = lane < PTH / 32 ? sh.red_s[lane] : -1.0;
            int i2 = lane < PTH / 32 ? sh.red_i[lane] : 0x7fffffff;
            warp_argmax(s2, i2);
            if (lane == 0) { sh.cand_score[par] = s2; sh.cand_row[par] = i2; }
        }
        __syncthreads();
        const int cr = sh.cand_row[par];
        if (tid < PW) {
            if (cr >= 0 && cr < N) {
                sh.cand_vals[par][0][tid] = Fr[at(cr, k0 + tid)];
                sh.cand_vals[par][1][tid] = Fi[at(cr, k0 + tid)];
            }
            if (c >= lo && c < hi) {
                sh.diag_vals[par][0][tid] = Fr[at(c, k0 + tid)];
                sh.diag_vals[par][1][tid] = Fi[at(c, k0 + tid)];
            }
        }
    };

    // initial candidates for column k0
    {
        double s = -1.0;
        int idx = 0x7fffffff;
        for (int r = max(lo, k0) + tid; r < hi; r += PTH) {
            double re = Fr[at(r, k0)], im = Fi[at(r, k0)];
            double sc = re * re + im * im;
            if (better(sc, r, s, idx)) { s = sc; idx = r; }
        }
        if (lo >= hi) idx = -1;
        publish(k0, 0, s, idx);
    }

    for (int jj = 0; jj < PW; ++jj) {
        const int j = k0 + jj;
        const int par = jj & 1;
        cluster.sync();
        if (wid == 0) {
            double s = -1.0;
            int idx = 0x7fffffff, win = 0;
            if (lane < PCL) {
                PanelShared* rs = cluster.map_shared_rank(&sh, lane);
                s = rs->cand_score[par];
                idx = rs->cand_row[par];
                if (idx < 0) { s = -1.0; idx = 0x7fffffff; }
            }
            int myrank = lane;
            // argmax carrying the owning rank
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                double so = __shfl_xor_sync(0xffffffffu, s, off);
                int io = __shfl_xor_sync(0xffffffffu, idx, off);
                int ro = __shfl_xor_sync(0xffffffffu, myrank, off);
                if (better(so, io, s, idx)) { s = so; idx = io; myrank = ro; }
            }
            win = myrank;
            if (lane == 0) {
                // all-zero column: Eigen keeps the diagonal row (no interchange)
                if (!(s > 0.0)) idx = j;
                sh.piv = idx;
                sh.winner = win;
            }
        }
        __syncthreads();
        const int piv = sh.piv;
        const int diag_owner = (j - k0) / R;
        if (tid < PW) {
            double ur, ui;
            if (piv == j) {
                PanelShared* ds = cluster.map_shared_rank(&sh, diag_owner);
                ur = ds->diag_vals[par][0][tid];
                ui = ds->diag_vals[par][1][tid];
            } else {
                PanelShared* ws = cluster.map_shared_rank(&sh, sh.winner);
                ur = ws->cand_vals[par][0][tid];
                ui = ws->cand_vals[par][1][tid];
                if (piv >= lo && piv < hi) {
                    // row piv receives the old row j
                    PanelShared* ds = cluster.map_shared_rank(&sh, diag_owner);
                    Fr[at(piv, k0 + tid)] = ds->diag_vals[par][0][tid];
                    Fi[at(piv, k0 + tid)] = ds->diag_vals[par][1][tid];
                }
                if (j >= lo && j < hi) {
                    Fr[at(j, k0 + tid)] = ur;
                    Fi[at(j, k0 + tid)] = ui;
                }
            }
            sh.u[0][tid] = ur;
            sh.u[1][tid] = ui;
        }
        if (rank == 0 && tid == 0) {
            ipiv[(long)b * N + j] = piv;
            sh.pivs[jj] = piv;
        }
        __syncthreads();
        // scale column j, rank-1 update of columns j+1..k0+63, candidates for j+1
        const cplx pv{sh.u[0][jj], sh.u[1][jj]};
        const bool nonzero = (pv.re != 0.0 || pv.im != 0.0);
        const cplx inv = nonzero ? crecip(pv) : cplx{0.0, 0.0};
        double s = -1.0;
        int idx = 0x7fffffff;
        for (int r = max(lo, j + 1) + tid; r < hi; r += PTH) {
            cplx l{Fr[at(r, j)], Fi[at(r, j)]};
            if (nonzero) {
                l = cmul(l, inv);
                Fr[at(r, j)] = l.re;
                Fi[at(r, j)] = l.im;
            }
            // chunks of 8 columns: all loads of a chunk are issued before any
            // store so the L2 round trips overlap (stores would otherwise
            // order every following load behind them)
            for (int c0 = jj + 1; c0 < PW; c0 += 8) {
                double xr[8], xi[8];
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (c0 + k < PW) {
                        xr[k] = Fr[at(r, k0 + c0 + k)];
                        xi[k] = Fi[at(r, k0 + c0 + k)];
                    }
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (c0 + k < PW) {
                        const double ur = sh.u[0][c0 + k], ui = sh.u[1][c0 + k];
                        xr[k] -= l.re * ur - l.im * ui;
                        xi[k] -= l.re * ui + l.im * ur;
                        Fr[at(r, k0 + c0 + k)] = xr[k];
                        Fi[at(r, k0 + c0 + k)] = xi[k];
                    }
                if (c0 == jj + 1) {
                    const double sc = xr[0] * xr[0] + xi[0] * xi[0];
                    if (better(sc, r, s, idx)) { s = sc; idx = r; }
                }
            }
        }
        if (jj + 1 < PW) {
            if (max(lo, j + 1) >= hi) idx = -1;
            __syncthreads();
            publish(j + 1, par ^ 1, s, idx);
        }
    }
    // rank 0: net permutation of the 64 interchanges (<= 128 rows move) for laswp
    if (rank == 0 && wid == 0) {
        for (int m = lane; m < PW; m += 32) {
            sh.tpos[m] = k0 + m;
            sh.tsrc[m] = k0 + m;
        }
        int cnt = PW;
        __syncwarp();
        for (int q = 0; q < PW; ++q) {
            const int pr = sh.pivs[q];
            if (pr == k0 + q) continue;
            int at_p;
            if (pr < k0 + PW) {
                at_p = pr - k0;
            } else {
                int hit = -1;
                for (int base = PW; base < cnt; base += 32) {
                    const int m = base + lane;
                    const unsigned bal = __ballot_sync(0xffffffffu, m < cnt && sh.tpos[m] == pr);
                    if (bal && hit < 0) hit = base + __ffs(bal) - 1;
                }
                if (hit < 0) {
                    hit = cnt;
                    if (lane == 0) {
                        sh.tpos[cnt] = pr;
                        sh.tsrc[cnt] = pr;
                    }
                    ++cnt;
                }
                at_p = hit;
            }
            __syncwarp();
            if (lane == 0) {
                const int t = sh.tsrc[q];
                sh.tsrc[q] = sh.tsrc[at_p];
                sh.tsrc[at_p] = t;
            }
            __syncwarp();
        }
        int* tab = ptab + (long)b * (4 * PW + 1);
        if (lane == 0) tab[0] = cnt;
        for (int m = lane; m < cnt; m += 32) {
            tab[1 + m] = sh.tpos[m];
            tab[1 + 2 * PW + m] = sh.tsrc[m];
        }
    }
    cluster.sync();  // keep shared memory alive until every CTA is done reading it
}

void launch_panel(ZBatch F, int N, int k0, int* ipiv, int* ptab, int batch, cudaStream_t s) {
    panel_kernel<<<dim3(PCL, batch), PTH, 0, s>>>(F, N, k0, ipiv, ptab);
}

// ------------------------------------------------------------------ laswp
// The panel's 64 interchanges applied to the columns outside the panel as one
// gather/scatter of the <= 128 moved rows (net permutation from the panel
// kernel): every load of a CTA is issued before any store.
constexpr int LS_COLS = 16;
__global__ void __launch_bounds__(256) laswp_panel_kernel(ZBatch F, int N, int k0,
                                                          const int* __restrict__ ptab) {
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
    const int ncols = N - PW;
    double* Fr = F.re + b * F.stride;
    double* Fi = F.im + b * F.stride;
    const int c0 = blockIdx.x * LS_COLS;
    for (int e = threadIdx.x; e < cnt * LS_COLS; e += blockDim.x) {
        const int m = e % cnt, c = e / cnt;
        int col = c0 + c;
        if (col >= ncols) continue;
        if (col >= k0) col += PW;
        const long o = (long)col * F.ld + src[m];
        vr[m][c] = Fr[o];
        vi[m][c] = Fi[o];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < cnt * LS_COLS; e += blockDim.x) {
        const int m = e % cnt, c = e / cnt;
        int col = c0 + c;
        if (col >= ncols) continue;
        if (col >= k0) col += PW;
        const long o = (long)col * F.ld + pos[m];
        Fr[o] = vr[m][c];
        Fi[o] = vi[m][c];
    }
}

void launch_laswp_panel(ZBatch F, int N, int k0, const int* ptab, int batch, cudaStream_t s) {
    const int ncols = N - PW;
    if (ncols <= 0) return;
    laswp_panel_kernel<<<dim3((ncols + LS_COLS - 1) / LS_COLS, batch), 256, 0, s>>>(F, N, k0, ptab);
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
    const long total = (long)N * P;
    for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long)gridDim.x * blockDim.x) {
        const long c = e / N, r = e - c * N;
        double y = add ? Y[c * ldy + r] : 0.0;
        for (int b = 0; b < batch; ++b) {
            const long o = b * W.stride + c * W.ld + r;
            const double t = __dsub_rn(__dmul_rn(w.zr[b], W.re[o]), __dmul_rn(w.zi[b], W.im[o]));
            y = __dadd_rn(y, t);
        }
        Y[c * ldy + r] = y;
    }
}

void launch_accumulate(ZBatch W, int N, int P, const NodeShifts& w, int batch, double* Y, long ldy,
                       bool add_to_Y, cudaStream_t s) {
    if (P <= 0) return;
    accumulate_kernel<<<148 * 4, 256, 0, s>>>(W, N, P, w, batch, Y, ldy, add_to_Y);
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
