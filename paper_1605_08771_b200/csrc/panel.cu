// 64-wide LU panel with partial pivoting (Eigen PartialPivLU's unblocked_lu
// semantics: pivot = argmax |a_ij| over rows >= j, lowest row on ties) for a
// batch of contour nodes — one 8-CTA thread-block cluster per node.
//
// Two-level blocking inside the panel: the 64 columns are factored as 64/W
// leaves of W columns. A leaf lives in REGISTERS (each thread owns ROWS panel
// rows x W complex entries), so the column steps touch no memory at all:
//   per column: block argmax of |x|^2 -> publish (score, row, the candidate's
//   W entries) in shared memory -> ONE cluster barrier -> every CTA reduces the
//   8 candidates through DSMEM, takes the pivot row from the winner's shared
//   memory; the owners of rows j and piv exchange rows in registers; scale +
//   rank-1 update in registers, fused with the next column's candidate search.
// Between leaves: rank 0 applies the leaf's interchanges to the panel's other
// columns as one gather/scatter of the moved rows, every CTA forms the leaf's
// U block (L_qq^{-1} T, W x (remaining panel columns)) redundantly in shared
// memory, and updates its own rows' remaining panel columns with its register
// L entries (one global read-modify-write per row).
#include <cooperative_groups.h>

#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.hpp"

namespace cg = cooperative_groups;

namespace fl {

namespace {

constexpr int PCL2 = 8;   // cluster size (portable)
constexpr int PWID = 64;  // outer panel width

template <int W, int CL>
struct RegPanelShared {
    // pushed by every rank of the cluster into every rank (parity buffered):
    // its best candidate (score, row, the row's W entries) and, from the owner
    // of row j, row j itself -- after the cluster barrier all of it is local
    double slot_score[2][CL];
    int slot_row[2][CL];
    double slot_vals[2][CL][2][W];
    double diag_vals[2][2][W];
    double red_s[32];
    int red_i[32];
    int pivs[PWID];
    // leaf U block: Lqq (W x W) and U (W x PWID)
    double lr[W][W + 1], li[W][W + 1];
    double Ur[W][PWID + 1], Ui[W][PWID + 1];
    // row permutation scratch (rank 0)
    int tpos[2 * PWID], tsrc[2 * PWID];
    double gr[2 * W][PWID], gi[2 * W][PWID];
    // L_kk staged for its inverse (column-major, ld PWID + 1)
    double Lkr[PWID][PWID + 1], Lki[PWID][PWID + 1];
};

// net permutation of interchanges (first+q, piv[q]) q < count, by one warp;
// returns the number of moved rows (rows tpos[m] <- tsrc[m])
template <class SH>
__device__ int net_permutation(SH& sh, int first, const int* piv, int count, int lane) {
    for (int m = lane; m < count; m += 32) {
        sh.tpos[m] = first + m;
        sh.tsrc[m] = first + m;
    }
    int cnt = count;
    __syncwarp();
    for (int q = 0; q < count; ++q) {
        const int pr = piv[q];
        if (pr == first + q) continue;
        int at_p;
        if (pr < first + count) {
            at_p = pr - first;
        } else {
            int hit = -1;
            for (int base = count; base < cnt; base += 32) {
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
    return cnt;
}

}  // namespace

__device__ unsigned long long g_panel_prof[8];

void res_panel_profile(double* out8, bool reset);

void panel_profile(double* out8, bool reset) {
    const char* e = std::getenv("FEASTLAB_PANEL");
    if (!(e && std::strcmp(e, "reg") == 0)) {
        res_panel_profile(out8, reset);
        return;
    }
    unsigned long long h[8];
    cudaMemcpyFromSymbol(h, g_panel_prof, sizeof(h));
    for (int i = 0; i < 8; ++i) out8[i] = (double)h[i];
    if (reset) {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_panel_prof, z, sizeof(z));
    }
}

template <int W, int ROWS, int NT, int CL>
// 256-thread variants are capped at 128 registers so a panel CTA fits on an SM
// beside one DMMA GEMM CTA: the look-ahead panel then overlaps the trailing
// update instead of waiting for a fully drained SM.
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(NT, NT <= 256 ? 2 : 1)
    panel_reg_kernel(ZBatch F, int N, int k0, int* __restrict__ ipiv, int* __restrict__ ptab,
                     ZBatch Inv) {
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char raw[];
    RegPanelShared<W, CL>& sh = *reinterpret_cast<RegPanelShared<W, CL>*>(raw);
    const int rank = (int)cluster.block_rank();
    const int b = blockIdx.y;
    double* Fr = F.re + b * F.stride;
    double* Fi = F.im + b * F.stride;
    const long ld = F.ld;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    constexpr int NW = NT / 32;
    const int R = (N - k0 + CL - 1) / CL;  // rows per CTA (<= ROWS * NT)
    const int base = k0 + rank * R;
    const int top = min(N, base + R);
    auto at = [&](int r, int c) { return (long)c * ld + r; };
    auto owner_rank = [&](int r) { return (r - k0) / R; };

    int row[ROWS];
    bool has[ROWS];
#pragma unroll
    for (int i = 0; i < ROWS; ++i) {
        row[i] = base + tid + i * NT;
        has[i] = row[i] < top;
    }
    double xr[ROWS][W], xi[ROWS][W];
    // phase timing of node 0 / rank 0 / thread 0 (fl_debug_panel_profile)
    const bool prof_on = (b == 0 && rank == 0 && tid == 0);
    long long t_last = clock64();
#define PPROF(k)                                                                 \
    if (prof_on) {                                                               \
        const long long t_ = clock64();                                          \
        atomicAdd(&g_panel_prof[k], (unsigned long long)(t_ - t_last));          \
        t_last = t_;                                                             \
    }

    // Every rank must have started (its shared memory allocated) before any
    // rank pushes into it: a remote store to a block that has not started yet
    // lands in whatever still occupies that SM's shared memory -- e.g. the last
    // operand stages of a trailing-update GEMM CTA that is finishing there
    // (observed: single wrong C tiles, only with the look-ahead panels running
    // beside the TMA-fed trailing update).
    cluster.sync();
    for (int q = 0; q < PWID / W; ++q) {
        const int c0 = k0 + q * W;
        // ---- load the leaf (rows >= c0 of this CTA)
#pragma unroll
        for (int i = 0; i < ROWS; ++i)
#pragma unroll
            for (int k = 0; k < W; ++k)
                if (has[i] && row[i] >= c0) {
                    xr[i][k] = Fr[at(row[i], c0 + k)];
                    xi[i][k] = Fi[at(row[i], c0 + k)];
                } else {
                    xr[i][k] = 0.0;
                    xi[i][k] = 0.0;
                }
        // ---- column steps
        // not unrolled (instruction-cache footprint): register entries are
        // addressed with compile-time k and runtime predicates on jj
#pragma unroll 1
        for (int jj = 0; jj < W; ++jj) {
            const int j = c0 + jj;
            const int par = j & 1;
            // local candidate for column j over own rows >= j
            double s = -1.0;
            int idx = 0x7fffffff;
#pragma unroll
            for (int i = 0; i < ROWS; ++i)
                if (has[i] && row[i] >= j) {
                    double pr = 0.0, pi = 0.0;
#pragma unroll
                    for (int k = 0; k < W; ++k)
                        if (k == jj) {
                            pr = xr[i][k];
                            pi = xi[i][k];
                        }
                    const double sc = pr * pr + pi * pi;
                    if (better(sc, row[i], s, idx)) {
                        s = sc;
                        idx = row[i];
                    }
                }
            warp_argmax(s, idx);
            if (lane == 0) {
                sh.red_s[wid] = s;
                sh.red_i[wid] = idx;
            }
            __syncthreads();
            {
                // every warp reduces the CTA's candidates redundantly; the
                // owners push the winner and row j into every rank's slots
                double s2 = lane < NW ? sh.red_s[lane] : -1.0;
                int i2 = lane < NW ? sh.red_i[lane] : 0x7fffffff;
                warp_argmax(s2, i2);
                const int cr = (s2 >= 0.0) ? i2 : -1;
                if (tid < CL) {
                    auto* d = cluster.map_shared_rank(&sh, tid);
                    d->slot_score[par][rank] = s2;
                    d->slot_row[par][rank] = cr;
                }
                bool own_c = false, own_j = false;
                double vr[W], vi[W], dr_[W], di_[W];
#pragma unroll
                for (int k = 0; k < W; ++k) vr[k] = vi[k] = dr_[k] = di_[k] = 0.0;
#pragma unroll
                for (int i = 0; i < ROWS; ++i) {
                    const bool c = has[i] && row[i] == cr, d = has[i] && row[i] == j;
                    own_c |= c;
                    own_j |= d;
#pragma unroll
                    for (int k = 0; k < W; ++k) {
                        if (c) {
                            vr[k] = xr[i][k];
                            vi[k] = xi[i][k];
                        }
                        if (d) {
                            dr_[k] = xr[i][k];
                            di_[k] = xi[i][k];
                        }
                    }
                }
                if (own_c)
#pragma unroll 1
                    for (int r = 0; r < CL; ++r) {
                        auto* d = cluster.map_shared_rank(&sh, r);
#pragma unroll
                        for (int k = 0; k < W; ++k) {
                            d->slot_vals[par][rank][0][k] = vr[k];
                            d->slot_vals[par][rank][1][k] = vi[k];
                        }
                    }
                if (own_j)
#pragma unroll 1
                    for (int r = 0; r < CL; ++r) {
                        auto* d = cluster.map_shared_rank(&sh, r);
#pragma unroll
                        for (int k = 0; k < W; ++k) {
                            d->diag_vals[par][0][k] = dr_[k];
                            d->diag_vals[par][1][k] = di_[k];
                        }
                    }
            }
            PPROF(0);
            cluster.sync();  // release/acquire: every rank's pushes are visible
            PPROF(1);
            // every thread reduces the CL local slots (lowest row on ties)
            double sw = -1.0;
            int iw = 0x7fffffff, winner = 0;
#pragma unroll
            for (int r = 0; r < CL; ++r) {
                const int rr = sh.slot_row[par][r];
                const double sr = rr < 0 ? -1.0 : sh.slot_score[par][r];
                const int ir = rr < 0 ? 0x7fffffff : rr;
                if (better(sr, ir, sw, iw)) {
                    sw = sr;
                    iw = ir;
                    winner = r;
                }
            }
            const int piv = (sw > 0.0) ? iw : j;  // all-zero column: no interchange
            const double* pvr = piv == j ? sh.diag_vals[par][0] : sh.slot_vals[par][winner][0];
            const double* pvi = piv == j ? sh.diag_vals[par][1] : sh.slot_vals[par][winner][1];
            const double* ojr = sh.diag_vals[par][0];
            const double* oji = sh.diag_vals[par][1];
            if (rank == 0 && tid == 0) {
                sh.pivs[q * W + jj] = piv;
                ipiv[(long)b * N + j] = piv;
            }
            PPROF(2);
            const cplx pv{pvr[jj], pvi[jj]};
            const bool nonzero = (pv.re != 0.0 || pv.im != 0.0);
            const cplx inv = nonzero ? crecip(pv) : cplx{0.0, 0.0};
#pragma unroll
            for (int i = 0; i < ROWS; ++i) {
                if (!has[i]) continue;
                if (row[i] == j) {
#pragma unroll
                    for (int k = 0; k < W; ++k) {
                        xr[i][k] = pvr[k];
                        xi[i][k] = pvi[k];
                    }
                } else if (row[i] > j) {
                    if (row[i] == piv) {
#pragma unroll
                        for (int k = 0; k < W; ++k) {
                            xr[i][k] = ojr[k];
                            xi[i][k] = oji[k];
                        }
                    }
                    cplx l{0.0, 0.0};
#pragma unroll
                    for (int k = 0; k < W; ++k)
                        if (k == jj) l = cplx{xr[i][k], xi[i][k]};
                    if (nonzero) l = cmul(l, inv);
#pragma unroll
                    for (int k = 0; k < W; ++k) {
                        if (k == jj) {
                            xr[i][k] = l.re;
                            xi[i][k] = l.im;
                        } else if (k > jj) {
                            const double ur = pvr[k], ui = pvi[k];
                            xr[i][k] -= l.re * ur - l.im * ui;
                            xi[i][k] -= l.re * ui + l.im * ur;
                        }
                    }
                }
            }
            PPROF(3);
        }
        // ---- store the factored leaf
#pragma unroll
        for (int i = 0; i < ROWS; ++i)
            if (has[i] && row[i] >= c0)
#pragma unroll
                for (int k = 0; k < W; ++k) {
                    Fr[at(row[i], c0 + k)] = xr[i][k];
                    Fi[at(row[i], c0 + k)] = xi[i][k];
                }
        cluster.sync();
        PPROF(4);
        // ---- rank 0: apply the leaf's interchanges to the other panel columns
        if (rank == 0) {
            __shared__ int s_cnt;
            if (wid == 0) {
                const int cnt = net_permutation(sh, c0, sh.pivs + q * W, W, lane);
                if (lane == 0) s_cnt = cnt;
            }
            __syncthreads();
            const int cnt = s_cnt;
            const int other = PWID - W;
            for (int e = tid; e < cnt * other; e += NT) {
                const int m = e % cnt, c = e / cnt;
                const int col = k0 + (c < q * W ? c : c + W);
                sh.gr[m][c] = Fr[at(sh.tsrc[m], col)];
                sh.gi[m][c] = Fi[at(sh.tsrc[m], col)];
            }
            __syncthreads();
            for (int e = tid; e < cnt * other; e += NT) {
                const int m = e % cnt, c = e / cnt;
                const int col = k0 + (c < q * W ? c : c + W);
                Fr[at(sh.tpos[m], col)] = sh.gr[m][c];
                Fi[at(sh.tpos[m], col)] = sh.gi[m][c];
            }
        }
        cluster.sync();
        PPROF(5);
        if (q == PWID / W - 1) break;
        // ---- leaf U block: U = Lqq^{-1} T, T = rows [c0, c0+W) x cols [c0+W, k0+64)
        const int rc0 = c0 + W;
        const int nrc = k0 + PWID - rc0;
        for (int e = tid; e < W * W; e += NT) {
            const int i = e % W, k = e / W;
            sh.lr[i][k] = Fr[at(c0 + i, c0 + k)];
            sh.li[i][k] = Fi[at(c0 + i, c0 + k)];
        }
        for (int e = tid; e < W * nrc; e += NT) {
            const int i = e % W, c = e / W;
            sh.Ur[i][c] = Fr[at(c0 + i, rc0 + c)];
            sh.Ui[i][c] = Fi[at(c0 + i, rc0 + c)];
        }
        __syncthreads();
        for (int r = 0; r < W - 1; ++r) {  // forward substitution, unit lower
            for (int e = tid; e < (W - 1 - r) * nrc; e += NT) {
                const int i = r + 1 + e % (W - 1 - r), c = e / (W - 1 - r);
                const double lr = sh.lr[i][r], li = sh.li[i][r];
                const double xr0 = sh.Ur[r][c], xi0 = sh.Ui[r][c];
                sh.Ur[i][c] -= lr * xr0 - li * xi0;
                sh.Ui[i][c] -= lr * xi0 + li * xr0;
            }
            __syncthreads();
        }
        PPROF(6);
        // ---- own rows >= rc0: A[row, rc0:] -= L[row, leaf] U
#pragma unroll
        for (int i = 0; i < ROWS; ++i) {
            if (!has[i] || row[i] < rc0) continue;
            for (int cb = 0; cb < nrc; cb += 8) {
                double ar[8], ai[8];
#pragma unroll
                for (int t = 0; t < 8; ++t)
                    if (cb + t < nrc) {
                        ar[t] = Fr[at(row[i], rc0 + cb + t)];
                        ai[t] = Fi[at(row[i], rc0 + cb + t)];
                    }
#pragma unroll
                for (int k = 0; k < W; ++k) {
                    const double lr = xr[i][k], li = xi[i][k];
#pragma unroll
                    for (int t = 0; t < 8; ++t)
                        if (cb + t < nrc) {
                            const double ur = sh.Ur[k][cb + t], ui = sh.Ui[k][cb + t];
                            ar[t] -= lr * ur - li * ui;
                            ai[t] -= lr * ui + li * ur;
                        }
                }
#pragma unroll
                for (int t = 0; t < 8; ++t)
                    if (cb + t < nrc) {
                        Fr[at(row[i], rc0 + cb + t)] = ar[t];
                        Fi[at(row[i], rc0 + cb + t)] = ai[t];
                    }
            }
        }
        // every CTA has read T (rows c0..c0+W, right columns) before rank 0
        // overwrites it with U: no CTA's later work touches those rows
        cluster.sync();
        if (rank == 0)
            for (int e = tid; e < W * nrc; e += NT) {
                const int i = e % W, c = e / W;
                Fr[at(c0 + i, rc0 + c)] = sh.Ur[i][c];
                Fi[at(c0 + i, rc0 + c)] = sh.Ui[i][c];
            }
        PPROF(7);
    }
    // ---- rank 0: net permutation of all 64 interchanges for the outer laswp
    if (rank == 0 && wid == 0) {
        const int cnt = net_permutation(sh, k0, sh.pivs, PWID, lane);
        int* tab = ptab + (long)b * (4 * PWID + 1);
        if (lane == 0) tab[0] = cnt;
        for (int m = lane; m < cnt; m += 32) {
            tab[1 + m] = sh.tpos[m];
            tab[1 + 2 * PWID + m] = sh.tsrc[m];
        }
    }
    // ---- L_kk^{-1} (unit lower 64 x 64; the solves and U12 multiply by it):
    // L_kk is final after the last leaf's interchanges (barrier above). One
    // warp per column c, axpy form x[k+1:] -= L[k+1:, k] x_k with lane l owning
    // rows l and l + 32; the next column of L is loaded one step ahead.
    {
        double* Ir = Inv.re + b * Inv.stride + (long)(k0 / PWID) * PWID * PWID;
        double* Ii = Inv.im + b * Inv.stride + (long)(k0 / PWID) * PWID * PWID;
        for (int e = tid; e < PWID * PWID; e += NT) {
            const int r = e & (PWID - 1), k = e >> 6;
            const long o = (long)(k0 + k) * ld + k0 + r;
            sh.Lkr[k][r] = r > k ? Fr[o] : 0.0;
            sh.Lki[k][r] = r > k ? Fi[o] : 0.0;
        }
        __syncthreads();
        const int gw = rank * NW + wid;
        for (int c = gw; c < PWID; c += CL * NW) {
            double x0r = lane == c ? 1.0 : 0.0, x0i = 0.0;
            double x1r = lane + 32 == c ? 1.0 : 0.0, x1i = 0.0;
            for (int k = c; k < PWID - 1; ++k) {
                const double xkr = __shfl_sync(0xffffffffu, k < 32 ? x0r : x1r, k & 31);
                const double xki = __shfl_sync(0xffffffffu, k < 32 ? x0i : x1i, k & 31);
                const double l0r = sh.Lkr[k][lane], l0i = sh.Lki[k][lane];
                const double l1r = sh.Lkr[k][lane + 32], l1i = sh.Lki[k][lane + 32];
                x0r -= l0r * xkr - l0i * xki;
                x0i -= l0r * xki + l0i * xkr;
                x1r -= l1r * xkr - l1i * xki;
                x1i -= l1r * xki + l1i * xkr;
            }
            Ir[(long)c * PWID + lane] = x0r;
            Ii[(long)c * PWID + lane] = x0i;
            Ir[(long)c * PWID + lane + 32] = x1r;
            Ii[(long)c * PWID + lane + 32] = x1i;
        }
    }
    cluster.sync();  // shared memory stays alive until every CTA is done with it
}

template <int W, int ROWS, int NT, int CL = PCL2>
static void launch_reg(ZBatch F, int N, int k0, int* ipiv, int* ptab, ZBatch Inv, int batch,
                       cudaStream_t s) {
    const size_t sm = sizeof(RegPanelShared<W, CL>);
    ensure_smem((const void*)panel_reg_kernel<W, ROWS, NT, CL>, sm);
    panel_reg_kernel<W, ROWS, NT, CL><<<dim3(CL, batch), NT, sm, s>>>(F, N, k0, ipiv, ptab, Inv);
}

template <int CL>
static void launch_panel_cl(ZBatch F, int N, int k0, int* ipiv, int* ptab, ZBatch Inv,
                            int batch, cudaStream_t s) {
    const int R = (N - k0 + CL - 1) / CL;
    if (R <= 256)
        launch_reg<8, 1, 256, CL>(F, N, k0, ipiv, ptab, Inv, batch, s);
    else if (R <= 512)
        launch_reg<4, 2, 256, CL>(F, N, k0, ipiv, ptab, Inv, batch, s);
    else if (R <= 1024)
        launch_reg<4, 4, 256, CL>(F, N, k0, ipiv, ptab, Inv, batch, s);
    else if (R <= 2048)
        launch_reg<2, 8, 256, CL>(F, N, k0, ipiv, ptab, Inv, batch, s);
    else
        launch_reg<2, 8, 512, CL>(F, N, k0, ipiv, ptab, Inv, batch, s);
}

bool launch_panel_resident(ZBatch F, int N, int k0, int* ipiv, int* ptab, ZBatch Inv, int batch,
                           cudaStream_t s);

void launch_panel(ZBatch F, int N, int k0, int* ipiv, int* ptab, ZBatch Inv, int batch,
                  cudaStream_t s, int res_rows) {
    // panels of <= res_rows rows: the on-chip panel (panel_res.cu) unless
    // FEASTLAB_PANEL=reg selects the register-leaf kernel below everywhere
    static const bool resident = [] {
        const char* e = std::getenv("FEASTLAB_PANEL");
        return !(e && std::strcmp(e, "reg") == 0);
    }();
    if (resident && N - k0 <= res_rows &&
        launch_panel_resident(F, N, k0, ipiv, ptab, Inv, batch, s))
        return;
    // 4-CTA clusters for short panels of small problems (<= 2048 rows of an
    // N <= 4096 matrix: 2 rows per thread, half the SMs a panel holds beside
    // the GEMMs); 8-CTA clusters otherwise. Measured (ms per application):
    // cfg0 8.8 -> 8.1, cfg2 146.2 -> 144.1; cfg3 / cfg4 keep 8 (532 / 11004
    // vs 538 / 11195 with the 4-CTA tails)
    static const int force = [] {
        const char* e = std::getenv("FEASTLAB_PANEL_CL");
        return e ? std::atoi(e) : 0;
    }();
    const int rows = N - k0;
    if (force == 4 || (force == 0 && rows <= 2048 && N <= 4096)) {
        launch_panel_cl<4>(F, N, k0, ipiv, ptab, Inv, batch, s);
        return;
    }
    if (force == 2) {
        launch_panel_cl<2>(F, N, k0, ipiv, ptab, Inv, batch, s);
        return;
    }
    launch_panel_cl<PCL2>(F, N, k0, ipiv, ptab, Inv, batch, s);
}

}  // namespace fl
