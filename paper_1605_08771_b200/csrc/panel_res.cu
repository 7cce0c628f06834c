// Latency-optimised 64-wide LU panel with partial pivoting (same semantics as
// panel.cu / Eigen PartialPivLU's unblocked_lu, proj/src/filterop.cpp:14:
// pivot = argmax |a_ij| over rows >= j, lowest row on ties, no interchange or
// scaling for an all-zero column) for panels of at most 4096 rows — the whole
// panel stays ON CHIP for the duration of the kernel.
//
// One thread-block cluster per node, CL = 1..16 CTAs of 256 threads; thread t
// of rank r owns panel row k0 + r*R + t (R = ceil(rows / CL) <= 256):
//   * the current leaf of W = 16 columns lives in its registers,
//   * the other three leaves live in shared memory (3 x 16 x 256 x 16 B =
//     192 KB; a leaf swaps registers <-> shared memory thread-locally),
// so HBM / L2 is touched once to load the panel and once to store it.
//
// Column step (the critical path), no cluster barrier:
//   exact warp argmax of |x|^2 as three REDUX ops -> CTA argmax of the 8 warp
//   winners (one __syncthreads, three REDUX) -> every CTA PUSHES its
//   candidate (key, row, 1/pivot, W values) and rank 0 the current diagonal
//   row into every rank's shared memory with st.async, each store completing
//   transaction bytes on the receiver's mbarrier (3 buffers in flight) ->
//   each CTA waits on its own mbarrier, reduces the CL keys (three REDUX) and
//   updates its rows. Look-ahead: a row updates only the next pivot column
//   at once; the rest of the rank-1 update runs while the next column's
//   exchange is in flight (pushers apply it to the row they send).
// Leaf transition (3 per panel): the leaf's interchanges as one net row
// permutation on the shared-memory columns (DSMEM gather, cluster barrier,
// scatter); rank 0 forms U = L_qq^{-1} T (one thread per column) and publishes
// it through global memory (it is final panel data); every CTA applies the
// rank-16 update to its shared-memory columns with its register L entries.
//
// Measured (B200, cfg2 n = 4096, one node): 64 panels 13 ms (register-leaf
// panel.cu: 27 ms); ~3k cycles per column step, bound by the dependent
// instruction chain of each warp (ncu: IPC 0.6, stall_wait/long_sb/mio), not
// by the DSMEM payload (halving it changed nothing).
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include <type_traits>

#include "common.cuh"
#include "kernels.hpp"

namespace cg = cooperative_groups;

namespace fl {

namespace {

constexpr int RW = 16;              // leaf width
constexpr int RNT = 256;            // threads per CTA = max rows per CTA
constexpr int RPW = 64;             // panel width
constexpr int NLEAF = RPW / RW;     // 4
constexpr int NSLOT = NLEAF - 1;    // leaves held in shared memory
constexpr int NWARP = RNT / 32;
constexpr int NBUF = 3;            // exchange buffers (columns in flight)
constexpr int PMAX = (2 * RW * (RPW - RW) + RNT - 1) / RNT;  // perm items per thread

template <int CL>
struct ResShared {
    double2 slot[NSLOT][RW][RNT];  // [slot][column][local row]
    // per-column exchange, buffered over 3 columns (written remotely by
    // st.async): a buffer is read up to one column after its own (the
    // deferred update), and a producer can run at most two columns ahead
    uint4 xhdr[NBUF][CL];          // {key hi, key lo, row, -} of every rank's candidate
    double2 xinv[NBUF][CL];        // 1 / (candidate's pivot entry)
    double2 xval[NBUF][CL][RW];    // the candidates' leaf values
    double2 xdiag[NBUF][RW];       // row j's leaf values (pushed by rank 0)
    uint64_t mbar[NBUF];
    // local staging, parity buffered
    double2 wval[2][NWARP][RW];    // each warp's winner row
    uint4 wkey[2][NWARP];          // each warp's winner key {hi, lo, row, -}
    double2 winv[2][NWARP];
    double2 dloc[2][RW];           // row j (rank 0)
    int pivs[RPW];
    int tpos[2 * RPW], tsrc[2 * RPW];
    int cnt;
    double2 lq[RW][RW];            // rank 0: L_qq
};

FL_DEV uint32_t mapa(uint32_t local, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}

// remote 16-byte store whose completion is counted (bytes) on the remote mbarrier
FL_DEV void st_async2(uint32_t raddr, double a, double b, uint32_t rbar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(
            raddr),
        "d"(a), "d"(b), "r"(rbar)
        : "memory");
}

FL_DEV void mbar_wait_cluster(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAITC_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAITC_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

FL_DEV void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// Exact argmax of a non-negative double score with ties to the lowest row,
// as three warp REDUX operations instead of a 5-level shuffle tree (a shuffle
// level costs ~80 cycles of latency on B200, a REDUX ~25). The key of a
// valid lane is (high word of the score's bits + 1, low word): for scores
// >= +0 the bit pattern is monotone; invalid lanes have key (0, 0). Returns
// the winning key in (hi, lo) and its row (0x7fffffff if no lane is valid).
FL_DEV int redux_argmax(unsigned& hi, unsigned& lo, int row, unsigned mask = 0xffffffffu) {
    const unsigned m1 = __reduce_max_sync(mask, hi);
    const unsigned m2 = __reduce_max_sync(mask, hi == m1 ? lo : 0u);
    const unsigned r = __reduce_min_sync(mask, (hi == m1 && lo == m2) ? (unsigned)row : 0x7fffffffu);
    hi = m1;
    lo = m2;
    return m1 == 0u ? 0x7fffffff : (int)r;
}

// f(integral_constant<int, jj>) for a warp-uniform runtime jj < 16: the leaf
// column is a compile-time register index inside f, while the code around
// the call is emitted once (a fully unrolled column loop overflows the
// instruction cache)
template <class F>
FL_DEV void dispatch16(int jj, F&& f) {
    switch (jj) {
#define FL_D16(J)                              \
    case J:                                    \
        f(std::integral_constant<int, J>{});   \
        break;
        FL_D16(0) FL_D16(1) FL_D16(2) FL_D16(3) FL_D16(4) FL_D16(5) FL_D16(6) FL_D16(7)
        FL_D16(8) FL_D16(9) FL_D16(10) FL_D16(11) FL_D16(12) FL_D16(13) FL_D16(14) FL_D16(15)
#undef FL_D16
        default:
            break;
    }
}

FL_DEV double ull_as_double(unsigned long long v) { return __longlong_as_double((long long)v); }

// x -= l * u (complex), one rounding per fma
FL_DEV void csub_mul(double2& x, double2 l, double2 u) {
    x.x = fma(-l.x, u.x, fma(l.y, u.y, x.x));
    x.y = fma(-l.x, u.y, fma(-l.y, u.x, x.y));
}

// net permutation of the interchanges (first+q, piv[q]) q < count, by one
// warp: rows tpos[m] <- tsrc[m] for m < return value
template <class SH>
FL_DEV int net_perm(SH& sh, int first, const int* piv, int count, int lane) {
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

__device__ unsigned long long g_res_prof[8];
__device__ long long g_res_trace[64 * 2 * 8 * 8];

int res_panel_trace(long long* out, int max) {
    const int n = max < 64 * 2 * 8 * 8 ? max : 64 * 2 * 8 * 8;
    cudaMemcpyFromSymbol(out, g_res_trace, sizeof(long long) * n);
    return n;
}

void res_panel_profile(double* out8, bool reset) {
    unsigned long long h[8];
    cudaMemcpyFromSymbol(h, g_res_prof, sizeof(h));
    for (int i = 0; i < 8; ++i) out8[i] = (double)h[i];
    if (reset) {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_res_prof, z, sizeof(z));
    }
}

template <int CL>
__global__ void __launch_bounds__(RNT, 1)
    panel_res_kernel(ZBatch F, int N, int k0, int* __restrict__ ipiv, int* __restrict__ ptab,
                     ZBatch Inv) {
    extern __shared__ __align__(16) unsigned char raw[];
    ResShared<CL>& sh = *reinterpret_cast<ResShared<CL>*>(raw);
    const int rank = CL > 1 ? (int)cg::this_cluster().block_rank() : 0;
    const int b = blockIdx.y;
    double* Fr = F.re + b * F.stride;
    double* Fi = F.im + b * F.stride;
    const long ld = F.ld;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int rows = N - k0;
    const int R = (rows + CL - 1) / CL;
    const int base = k0 + rank * R;
    const int row = base + tid;
    const bool own = tid < R && row < N;
    auto at = [&](int r, int c) { return (long)c * ld + r; };
#ifdef FL_PANEL_PROF
    // phase timing of node 0 / rank 0 / thread 0 (fl_debug_panel_profile;
    // build with EXTRA=-DFL_PANEL_PROF)
    const bool prof_on = (b == 0 && rank == 0 && lane == 0);  // summed over the 8 warps
    long long t_last = clock64();
#define RPROF(k)                                                                 \
    if (prof_on) {                                                               \
        const long long t_ = clock64();                                          \
        atomicAdd(&g_res_prof[k], (unsigned long long)(t_ - t_last));            \
        t_last = t_;                                                             \
    }
#else
#define RPROF(k)
#endif
#ifdef FL_PANEL_TRACE
    // clock64 of lane 0 of every warp of ranks 0 and CL-1 at 4 points of every
    // column of the first panel (k0 == 0) of node 0 (fl_debug_panel_trace)
#define RTRACE(tag)                                                                        \
    if (b == 0 && (rank == 0 || rank == CL - 1) && lane == 0 && k0 == 0)                   \
        g_res_trace[(((jl * 2 + (rank != 0)) * NWARP + wid) * 8) + (tag)] = clock64();
#else
#define RTRACE(tag)
#endif

    // ---- load the panel: leaf 0 -> registers, leaves 1..3 -> slots 0..2
    double2 x[RW];
#pragma unroll
    for (int k = 0; k < RW; ++k)
        x[k] = own ? make_double2(Fr[at(row, k0 + k)], Fi[at(row, k0 + k)]) : make_double2(0, 0);
#pragma unroll
    for (int s = 0; s < NSLOT; ++s)
#pragma unroll
        for (int k = 0; k < RW; ++k) {
            const int c = k0 + RW * (s + 1) + k;
            sh.slot[s][k][tid] = own ? make_double2(Fr[at(row, c)], Fi[at(row, c)])
                                     : make_double2(0, 0);
        }
    if (tid == 0) {
#pragma unroll
        for (int i = 0; i < NBUF; ++i) mbar_init(&sh.mbar[i], 1);
        mbar_fence_init();
    }
    if (CL > 1) cluster_sync_all(); else __syncthreads();
    RPROF(0);

    const uint32_t xhdr0 = smem_u32(&sh.xhdr[0][0]);
    const uint32_t xval0 = smem_u32(&sh.xval[0][0][0]);
    const uint32_t xdiag0 = smem_u32(&sh.xdiag[0][0]);
    const uint32_t xinv0 = smem_u32(&sh.xinv[0][0]);
    const uint32_t mbar0 = smem_u32(&sh.mbar[0]);
    constexpr unsigned kBytes = CL * (RW + 2) * 16 + RW * 16;  // per column, per receiver

    for (int q = 0; q < NLEAF; ++q) {
        const int c0 = k0 + q * RW;
        // ---------------------------------------------------------- column steps
        // Unrolled: the leaf column jj is a compile-time register index.
        // Look-ahead by one column: after the exchange of column jj a row
        // updates only entry jj+1 at once (the next pivot column) and
        // applies the rest of column jj's rank-1 update (entries >= jj+2)
        // while the exchange of column jj+1 is in flight. A candidate row is
        // therefore pushed with that pending update applied by the pusher.
        // l_prev / pend: this row's multiplier of the previous column and
        // whether a deferred update is pending for it.
        double2 l_prev = make_double2(0, 0);
        bool pend = false;
        const double2* ppv = sh.xdiag[0];  // previous column's pivot row (smem)
#pragma unroll 1
        for (int jj = 0; jj < RW; ++jj) {
            const int jl = q * RW + jj;
            const int j = k0 + jl;
            const int par = jl & 1;
            const int bf = jl % NBUF;  // exchange buffer of this column
            RTRACE(0);
            const bool valid = own && row >= j;
            double2 xj;
            dispatch16(jj, [&](auto c) { xj = x[decltype(c)::value]; });
            const double sc = xj.x * xj.x + xj.y * xj.y;
            // reciprocal of the own pivot candidate, off the critical path
            // (overlaps the reductions); only the winner's is used. Rows that
            // cannot win divide a dummy 1: a zero or non-finite divisor would
            // take the division's slow path and stall the whole warp.
            const double rs = 1.0 / ((valid && sc > 0.0 && sc < 1e300) ? sc : 1.0);
            const double2 myinv = make_double2(xj.x * rs, -xj.y * rs);
            const unsigned long long bits = (unsigned long long)__double_as_longlong(sc);
            unsigned hi = valid ? (unsigned)(bits >> 32) + 1u : 0u;
            unsigned lo = valid ? (unsigned)bits : 0u;
            if (rank == 0 && row == j) {  // the diagonal row, for rank 0's push
#pragma unroll
                for (int k = 0; k < RW; ++k) sh.dloc[par][k] = x[k];
            }
            const int wr = redux_argmax(hi, lo, row);
            if (row == wr) {
#pragma unroll
                for (int k = 0; k < RW; ++k) sh.wval[par][wid][k] = x[k];
                sh.winv[par][wid] = myinv;
            }
            if (lane == 0) sh.wkey[par][wid] = make_uint4(hi, lo, (unsigned)wr, 0u);
            RPROF(1);
            RTRACE(1);
            __syncthreads();
            RTRACE(2);
            // CTA candidate: every warp reduces the warps' winners (lanes < 8)
            unsigned chi = 0u, clo = 0u;
            int crow = 0x7fffffff;
            if (lane < NWARP) {
                const uint4 kk = sh.wkey[par][lane];
                chi = kk.x;
                clo = kk.y;
                crow = (int)kk.z;
            }
            crow = redux_argmax(chi, clo, crow);
            const int wc = chi ? ((crow - base) >> 5) : 0;
            RPROF(2);
            RTRACE(5);
            // push: thread (r, k) sends value k of the candidate (and, on rank
            // 0, of row j) to rank r; threads r < CL send the key and 1/pivot.
            // Entries >= jj+1 still lack the previous column's update: the
            // pusher applies it (its row's multiplier is entry jj-1).
            {
                const unsigned bar = mbar0 + (unsigned)(bf * 8);
                if (tid < CL * RW) {
                    const int r = tid / RW, k = tid % RW;
                    const uint32_t rb = mapa(bar, r);
                    double2 v = sh.wval[par][wc][k];
                    double2 d = sh.dloc[par][k];
                    if (jj > 0 && k > jj) {
                        const double2 u = ppv[k];
                        csub_mul(v, sh.wval[par][wc][jj - 1], u);
                        csub_mul(d, sh.dloc[par][jj - 1], u);
                    }
                    st_async2(mapa(xval0 + (unsigned)(((bf * CL + rank) * RW + k) * 16), r), v.x,
                              v.y, rb);
                    if (rank == 0)
                        st_async2(mapa(xdiag0 + (unsigned)((bf * RW + k) * 16), r), d.x, d.y, rb);
                }
                if (tid < CL) {
                    const uint32_t rb = mapa(bar, tid);
                    st_async2(mapa(xhdr0 + (unsigned)((bf * CL + rank) * 16), tid),
                              ull_as_double(((unsigned long long)clo << 32) | chi),
                              ull_as_double((unsigned long long)(unsigned)crow), rb);
                    const double2 iv = sh.winv[par][wc];
                    st_async2(mapa(xinv0 + (unsigned)((bf * CL + rank) * 16), tid), iv.x, iv.y, rb);
                }
            }
            if (tid == 0) mbar_arrive_expect_tx(&sh.mbar[bf], kBytes);
            RPROF(3);
            RTRACE(6);
            // the previous column's deferred update (entries >= jj+1), in the
            // shadow of this column's exchange
            if (pend) {
                dispatch16(jj, [&](auto c) {
                    constexpr int J = decltype(c)::value;
#pragma unroll
                    for (int k = J + 1; k < RW; ++k) csub_mul(x[k], l_prev, ppv[k]);
                });
            }
            RPROF(4);
            RTRACE(3);
            mbar_wait_cluster(&sh.mbar[bf], (jl / NBUF) & 1);
            RTRACE(4);
            RPROF(5);
            // every warp reduces the CL candidates (lowest row on ties)
            unsigned ghi = 0u, glo = 0u;
            int hrow = 0x7fffffff;
            if (lane < CL) {
                const uint4 kk = sh.xhdr[bf][lane];
                ghi = kk.x;
                glo = kk.y;
                hrow = (int)kk.z;
            }
            const int grow = redux_argmax(ghi, glo, hrow);
            // rank holding the winner: the lane whose header carried its row
            const int wrk = max(0, __ffs(__ballot_sync(0xffffffffu, lane < CL && hrow == grow)) - 1);
            // winner score > 0 (key (1, 0) is +0.0): else no interchange
            const bool nonzero = ghi > 1u || (ghi == 1u && glo != 0u);
            const int piv = nonzero ? grow : j;
            if (tid == 0) {
                sh.pivs[jl] = piv;
                if (rank == 0) ipiv[(long)b * N + j] = piv;
            }
            const double2* pvv = piv == j ? sh.xdiag[bf] : sh.xval[bf][wrk];
            const double2 inv = nonzero ? sh.xinv[bf][wrk] : make_double2(0, 0);
            ppv = pvv;
            pend = false;
            if (own) {
                if (row == j) {
#pragma unroll
                    for (int k = 0; k < RW; ++k) x[k] = pvv[k];
                } else if (row > j) {
                    if (row == piv) {
#pragma unroll
                        for (int k = 0; k < RW; ++k) x[k] = sh.xdiag[bf][k];
                    }
                    dispatch16(jj, [&](auto c) {
                        constexpr int J = decltype(c)::value;
                        double2 l = x[J];
                        if (nonzero) {
                            const cplx m = cmul(cplx{l.x, l.y}, cplx{inv.x, inv.y});
                            l = make_double2(m.re, m.im);
                        }
                        x[J] = l;
                        if constexpr (J + 1 < RW) csub_mul(x[J + 1], l, pvv[J + 1]);
                        l_prev = l;
                    });
                    pend = jj + 2 < RW;
                }
            }
            RPROF(6);
        }
        // ---------------------------------------------------------- leaf transition
        // (1) the leaf's interchanges on the shared-memory columns (all slots)
        if (wid == 0) {
            const int cnt = net_perm(sh, c0, sh.pivs + q * RW, RW, lane);
            if (lane == 0) sh.cnt = cnt;
        }
        __syncthreads();
        const int cnt = sh.cnt;
        {
            constexpr int NC = NSLOT * RW;  // 48 shared-memory columns
            double2 buf[PMAX];
#pragma unroll
            for (int u = 0; u < PMAX; ++u) {
                const int it = tid + u * RNT;
                buf[u] = make_double2(0, 0);
                if (it < cnt * NC) {
                    const int m = it % cnt, c = it / cnt;
                    const int dst = sh.tpos[m];
                    if ((dst - k0) / R == rank) {
                        const int src = sh.tsrc[m];
                        const int sr = (src - k0) / R, sl = src - (k0 + sr * R);
                        const double2* p = &sh.slot[c / RW][c % RW][sl];
                        if (CL > 1 && sr != rank)
                            p = cg::this_cluster().map_shared_rank(const_cast<double2*>(p), sr);
                        buf[u] = *p;
                    }
                }
            }
            if (CL > 1) cluster_sync_all(); else __syncthreads();
#pragma unroll
            for (int u = 0; u < PMAX; ++u) {
                const int it = tid + u * RNT;
                if (it < cnt * NC) {
                    const int m = it % cnt, c = it / cnt;
                    const int dst = sh.tpos[m];
                    if ((dst - k0) / R == rank) sh.slot[c / RW][c % RW][dst - base] = buf[u];
                }
            }
        }
        __syncthreads();
        RPROF(7);
        if (q == NLEAF - 1) break;
        // (2) rank 0: U = L_qq^{-1} T on the remaining columns (slots q..2),
        // rows c0..c0+15, in place; published to global memory (final data)
        const int nrem = RPW - RW * (q + 1);
        if (rank == 0) {
            const int li = row - c0;
            if (li >= 0 && li < RW) {
#pragma unroll
                for (int k = 0; k < RW; ++k) sh.lq[li][k] = x[k];
            }
            __syncthreads();
            if (tid < nrem) {
                const int c = tid;
                const int sidx = q + c / RW, kc = c % RW;
                const int l0 = c0 - k0;
                double2 t[RW];
#pragma unroll
                for (int i = 0; i < RW; ++i) t[i] = sh.slot[sidx][kc][l0 + i];
#pragma unroll
                for (int r = 0; r < RW - 1; ++r)
#pragma unroll
                    for (int i = r + 1; i < RW; ++i) csub_mul(t[i], sh.lq[i][r], t[r]);
                const int col = c0 + RW + c;
#pragma unroll
                for (int i = 0; i < RW; ++i) {
                    sh.slot[sidx][kc][l0 + i] = t[i];
                    Fr[at(c0 + i, col)] = t[i].x;
                    Fi[at(c0 + i, col)] = t[i].y;
                }
            }
        }
        if (CL > 1) cluster_sync_all(); else __syncthreads();
        RPROF(7);
        // (3) rank-16 update of the own rows below the leaf's diagonal block;
        // U is read from global memory through L1 (one 128-byte line per
        // column and plane, shared by every thread of the CTA)
        if (own && row >= c0 + RW) {
            for (int c = 0; c < nrem; ++c) {
                const double* ur = Fr + at(c0, c0 + RW + c);
                const double* ui = Fi + at(c0, c0 + RW + c);
                double2& y = sh.slot[q + c / RW][c % RW][tid];
                double2 v = y;
#pragma unroll
                for (int k = 0; k < RW; ++k) csub_mul(v, x[k], make_double2(__ldca(ur + k), __ldca(ui + k)));
                y = v;
            }
        }
        // (4) leaf q -> slot q, leaf q+1 -> registers (thread-local)
#pragma unroll
        for (int k = 0; k < RW; ++k) {
            const double2 t = sh.slot[q][k][tid];
            sh.slot[q][k][tid] = x[k];
            x[k] = t;
        }
        RPROF(7);
        // no barrier: the next leaf's exchanges touch only the exchange
        // buffers, and every CTA's next remote slot access (the next
        // transition's gather) follows exchanges that this CTA completes
        // after finishing this transition
    }
    // ---- store the panel: slots 0..2 = leaves 0..2, registers = leaf 3
    if (own) {
#pragma unroll
        for (int s = 0; s < NSLOT; ++s)
#pragma unroll
            for (int k = 0; k < RW; ++k) {
                const double2 v = sh.slot[s][k][tid];
                Fr[at(row, k0 + RW * s + k)] = v.x;
                Fi[at(row, k0 + RW * s + k)] = v.y;
            }
#pragma unroll
        for (int k = 0; k < RW; ++k) {
            Fr[at(row, k0 + RW * NSLOT + k)] = x[k].x;
            Fi[at(row, k0 + RW * NSLOT + k)] = x[k].y;
        }
    }
    // ---- rank 0: net permutation of all 64 interchanges for the outer laswp
    if (rank == 0 && wid == 0) {
        const int cn = net_perm(sh, k0, sh.pivs, RPW, lane);
        int* tab = ptab + (long)b * (4 * RPW + 1);
        if (lane == 0) tab[0] = cn;
        for (int m = lane; m < cn; m += 32) {
            tab[1 + m] = sh.tpos[m];
            tab[1 + 2 * RPW + m] = sh.tsrc[m];
        }
    }
    if (CL > 1) cluster_sync_all(); else __syncthreads();  // L_kk in global, visible
    // ---- L_kk^{-1} (unit lower 64 x 64), one warp per column, staged in the
    // (now free) slot storage
    {
        double(*Lkr)[RPW + 1] = reinterpret_cast<double(*)[RPW + 1]>(&sh.slot[0][0][0]);
        double(*Lki)[RPW + 1] = Lkr + RPW;
        double* Ir = Inv.re + b * Inv.stride + (long)(k0 / RPW) * RPW * RPW;
        double* Ii = Inv.im + b * Inv.stride + (long)(k0 / RPW) * RPW * RPW;
        for (int e = tid; e < RPW * RPW; e += RNT) {
            const int r = e & (RPW - 1), k = e >> 6;
            const long o = (long)(k0 + k) * ld + k0 + r;
            Lkr[k][r] = r > k ? __ldcg(Fr + o) : 0.0;
            Lki[k][r] = r > k ? __ldcg(Fi + o) : 0.0;
        }
        __syncthreads();
        const int gw = rank * NWARP + wid;
        for (int c = gw; c < RPW; c += CL * NWARP) {
            double x0r = lane == c ? 1.0 : 0.0, x0i = 0.0;
            double x1r = lane + 32 == c ? 1.0 : 0.0, x1i = 0.0;
            for (int k = c; k < RPW - 1; ++k) {
                const double xkr = __shfl_sync(0xffffffffu, k < 32 ? x0r : x1r, k & 31);
                const double xki = __shfl_sync(0xffffffffu, k < 32 ? x0i : x1i, k & 31);
                const double l0r = Lkr[k][lane], l0i = Lki[k][lane];
                const double l1r = Lkr[k][lane + 32], l1i = Lki[k][lane + 32];
                x0r -= l0r * xkr - l0i * xki;
                x0i -= l0r * xki + l0i * xkr;
                x1r -= l1r * xkr - l1i * xki;
                x1i -= l1r * xki + l1i * xkr;
            }
            Ir[(long)c * RPW + lane] = x0r;
            Ii[(long)c * RPW + lane] = x0i;
            Ir[(long)c * RPW + lane + 32] = x1r;
            Ii[(long)c * RPW + lane + 32] = x1i;
        }
    }
    if (CL > 1) cluster_sync_all();
    RPROF(0);
#undef RPROF
}

template <int CL>
static void launch_res(ZBatch F, int N, int k0, int* ipiv, int* ptab, ZBatch Inv, int batch,
                       cudaStream_t s) {
    const size_t sm = sizeof(ResShared<CL>);
    static_assert(sizeof(ResShared<CL>) <= 232448, "panel_res shared memory");
    static_assert(2 * RPW * (RPW + 1) * sizeof(double) <= sizeof(double2) * NSLOT * RW * RNT,
                  "L_kk staging must fit the slot storage");
    auto kern = panel_res_kernel<CL>;
    // per device (a process may drive several GPUs: solve_concurrently)
    ensure_smem((const void*)kern, sm);
    if (CL > 8) ensure_attr((const void*)kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL, batch);
    cfg.blockDim = dim3(RNT);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    launch_check(cudaLaunchKernelEx(&cfg, kern, F, N, k0, ipiv, ptab, Inv), "panel_res launch");
}

// Resident panel for rows = N - k0 <= 4096: the smallest cluster whose CTAs
// hold at most 256 rows each. Returns false when the panel is too tall.
bool launch_panel_resident(ZBatch F, int N, int k0, int* ipiv, int* ptab, ZBatch Inv, int batch,
                           cudaStream_t s) {
    const int rows = N - k0;
    if (rows <= 256) launch_res<1>(F, N, k0, ipiv, ptab, Inv, batch, s);
    else if (rows <= 512) launch_res<2>(F, N, k0, ipiv, ptab, Inv, batch, s);
    else if (rows <= 1024) launch_res<4>(F, N, k0, ipiv, ptab, Inv, batch, s);
    else if (rows <= 2048) launch_res<8>(F, N, k0, ipiv, ptab, Inv, batch, s);
    else if (rows <= 4096) launch_res<16>(F, N, k0, ipiv, ptab, Inv, batch, s);
    else return false;
    return true;
}

}  // namespace fl
