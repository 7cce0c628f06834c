// Device-side implementation of the C ABI (include/feastlab_b200.h): contexts,
// device-resident matrices and blocks, the filter orchestration
// (FilterApplier::apply, proj/src/filterop.cpp:62-84) and the Rayleigh-Ritz
// sequence (proj/src/ritz.cpp:17-122) on the sm_100a kernels.
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/feastlab_b200.h"
#include "common.cuh"
#include "kernels.hpp"
#include "ritz_kernels.hpp"

namespace fl {
std::atomic<long long> g_launch_count{0};
}
// fl_debug_decision_log: the rounding-sensitive decisions of the drivers are
// written to stderr with their margins (tests/test_gpu_configs.py reads them)
static std::atomic<int> g_decision_log{0};

namespace {

using namespace fl;

inline int round_up(int x, int m) { return (x + m - 1) / m * m; }
constexpr int FL_MAX_BLOCK_PANELS = 16;  // LU outer block; solve row blocks <= 8

struct Fail {
    int code;
    std::string msg;
    int index = -1;
    double pivot = 0, zr = 0, zi = 0;
};

int report(fl_err* e, const Fail& f) {
    if (e) {
        e->status = f.code;
        e->index = f.index;
        e->pivot = f.pivot;
        e->z_re = f.zr;
        e->z_im = f.zi;
        std::snprintf(e->msg, sizeof(e->msg), "%s", f.msg.c_str());
    }
    return f.code;
}

void cuda_check(cudaError_t c, const char* what) {
    if (c != cudaSuccess) {
        if (c == cudaErrorMemoryAllocation)
            throw Fail{FL_OOM, std::string(what) + ": " + cudaGetErrorString(c)};
        throw Fail{FL_CUDA, std::string(what) + ": " + cudaGetErrorString(c)};
    }
}
#define CK(x) cuda_check((x), #x)

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw Fail{FL_NCCL, std::string(what) + ": " + ncclGetErrorString(r)};
}

// device allocation with RAII
struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    void ensure(size_t b) {
        if (b <= bytes) return;
        release();
        CK(cudaMalloc(&p, b));
        bytes = b;
    }
    double* d() const { return static_cast<double*>(p); }
    int* i() const { return static_cast<int*>(p); }
};

// Per-kernel-class CUDA-event timing (fl_ctx_set_profiling): bench.py's
// roofline numbers come from these events, recorded on the launch stream.
enum ProfClass { P_SHIFT, P_PANEL, P_LASWP, P_TRSM, P_ZGEMM, P_PERMUTE, P_ACCUM, P_ALLREDUCE,
                 P_EIG, P_ORTH, P_RR, P_ZSUM, P_NCLASS };
const char* const kProfNames[P_NCLASS] = {"shift",   "panel",      "laswp",    "trsm",
                                          "zgemm",   "permute",    "accumulate", "allreduce",
                                          "eig",     "orthonormalize", "rayleigh_ritz", "zsum"};

struct Profiler {
    struct Rec {
        int cls;
        cudaEvent_t a, b;
        double work;
        double tag;  // launch shape (zgemm classes: shape_tag), 0 otherwise
    };
    bool on = false;
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    cudaEvent_t get() {
        if (used == pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            pool.push_back(e);
        }
        return pool[used++];
    }
    void reset() {
        recs.clear();
        used = 0;
    }
    ~Profiler() {
        for (cudaEvent_t e : pool) cudaEventDestroy(e);
    }
};

}  // namespace

struct fl_filter;

struct fl_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int rank = 0, nranks = 1;
    ncclComm_t comm = nullptr;
    std::recursive_mutex mu;
    // the owner's reference plus one per live matrix / block / filter: a
    // context outlives its objects whatever order callers (or a garbage
    // collector breaking a reference cycle) destroy them in
    std::atomic<int> refs{1};
    long long launches_at_create = 0;
    Profiler prof;
    std::vector<cudaStream_t> aux;  // node-chunk streams (fork/join on `stream`)
    cudaEvent_t fork = nullptr;
    cudaEvent_t done = nullptr;  // host waits: polled (see sync())
    unsigned long long* h_cnt = nullptr;  // pinned: eigensolver sweep counter
    // filters whose singular-node flag is in flight (resolved by sync())
    std::vector<fl_filter*> pending;
    std::vector<cudaEvent_t> join;
    std::vector<cudaStream_t> paux;  // per chunk: look-ahead panel stream (high priority)
    std::vector<cudaEvent_t> ev_panel, ev_next;
    int nstreams = 8;  // node chunks in flight (<= aux.size())
    int reduction = 0;  // FL_REDUCE_SUM / FL_REDUCE_ORDERED (multi-rank Y)
    int factorization = 0;  // FL_FACTOR_LU / FL_FACTOR_LDLT
    // Rayleigh-Ritz scratch
    DBuf rr_nxp, rr_nxp2, s1, s2, s3, s4, s5, s6, s7, vals_d, norms_d, idx_d, chol_info, ints, cnt,
        scal;
};

struct fl_matrix {
    fl_ctx* ctx;
    int n, N;
    DBuf buf;
    double* d() const { return buf.d(); }
};

struct fl_block {
    fl_ctx* ctx;
    int n, N;
    int cols = 0, cap = 0, CAP = 0;
    int dirty = 0;  // columns [cols, dirty) may hold stale data
    DBuf buf;
    double* d() const { return buf.d(); }
    long ld() const { return N; }
};

struct fl_filter {
    fl_ctx* ctx;
    const fl_matrix* A;
    int nc;
    std::vector<double> zr, zi, wr, wi;
    bool cache;
    int kb = 0, ke = 0;  // local node range [kb, ke)
    // factors: cache -> one per local node; else a rotating group
    DBuf fac_re, fac_im, ipiv, perm, bad, ptab;
    DBuf cmap, btab;             // composed outer-block interchanges (launch_laswp_block)
    int laswp_block = 1;         // FEASTLAB_LASWP_BLOCK=0: one interchange pass per panel
    DBuf inv_re, inv_im;  // per slot: NB inverted L_ii blocks, then NB inverted U_ii blocks
    DBuf lt_re, lt_im;    // LDL^T: per slot, the current panel's L_kk^{-T} (64 x 64)
    // TMA-fed trailing updates (gemm_tma.cu): per slot the sum planes Re + Im of
    // the current outer block's L21 (N x sum_kb, ld N) and U12 (sum_kb x N, ld
    // sum_kb), and the tensor maps of the factor planes and the sum planes
    DBuf sum_a, sum_b;
    int sum_kb = 0;
    ZGemmMaps maps;
    bool maps_ok = false;
    int fac_mode = -1;    // factorization the cached factors were built with
    int fac_slots = 0;
    int panel_res_rows = 4096;   // see panel_res_rows()
    int lu_panels = 2;           // LU outer block = lu_panels x 64 columns (block_panels())
    int solve_panels = 4;        // triangular-solve row block = solve_panels x 64 rows
    std::vector<char> factored;  // cache mode, per local node
    DBuf w_re, w_im;             // W for all local nodes (N x P each)
    long w_stride = 0;
    int w_P = 0;
    DBuf y_tmp;
    DBuf terms, terms_all;  // ordered reduction: local / gathered Re(w_k W_k)
    // CUDA graph of one whole application (non-cache mode): captured on the
    // second call with an unchanged launch key, replayed while it holds
    struct GraphKey {
        const void *X, *Y, *fac, *w;
        long ldx, ldy;
        int p, slots, ns, zmode, reduction, factorization;
        int phase;  // 0: factor + solve (no cache); cache: 1 factor + solve, 2 solve only
        int lu_panels, solve_panels, panel_res_rows;  // blocking (environment-tunable)
        int laswp_block;
        bool operator==(const GraphKey& o) const {
            return X == o.X && Y == o.Y && fac == o.fac && w == o.w && ldx == o.ldx &&
                   ldy == o.ldy && p == o.p && slots == o.slots && ns == o.ns &&
                   zmode == o.zmode && reduction == o.reduction &&
                   factorization == o.factorization && phase == o.phase &&
                   lu_panels == o.lu_panels && solve_panels == o.solve_panels &&
                   panel_res_rows == o.panel_res_rows && laswp_block == o.laswp_block;
        }
    };
    GraphKey gkey{}, gseen{};
    cudaGraphExec_t gexec = nullptr;
    long long glaunches = 0;
    // first singular node of the last application (0x7f7f7f7f: none), copied
    // to pinned memory asynchronously and checked at the next host wait
    int* h_bad = nullptr;
    bool check_pending = false;
    ~fl_filter() {
        if (gexec) cudaGraphExecDestroy(gexec);
        if (h_bad) cudaFreeHost(h_bad);
    }
};

namespace {

struct CtxLock {
    std::lock_guard<std::recursive_mutex> lk;
    explicit CtxLock(fl_ctx* c) : lk(c->mu) { cudaSetDevice(c->device); }
};

void zero_cols(fl_block* b, int from, int to) {
    if (to > from)
        CK(cudaMemsetAsync(b->d() + (long)from * b->ld(), 0,
                           sizeof(double) * (size_t)b->ld() * (to - from), b->ctx->stream));
}

void block_set_cols(fl_block* b, int k) {
    // invariant: columns [cols, CAP) are zero
    if (b->dirty > k) zero_cols(b, k, b->dirty);
    b->cols = k;
    b->dirty = k;
}

void block_reserve(fl_block* b, int cap) {
    if (cap <= b->cap) return;
    const int CAP = round_up(std::max(cap, 1), FL_TILE);
    DBuf nb;
    nb.ensure(sizeof(double) * (size_t)b->N * CAP);
    CK(cudaMemsetAsync(nb.p, 0, sizeof(double) * (size_t)b->N * CAP, b->ctx->stream));
    if (b->cols > 0)
        CK(cudaMemcpyAsync(nb.p, b->buf.p, sizeof(double) * (size_t)b->N * b->cols,
                           cudaMemcpyDeviceToDevice, b->ctx->stream));
    std::swap(b->buf.p, nb.p);
    std::swap(b->buf.bytes, nb.bytes);
    b->cap = cap;
    b->CAP = CAP;
    b->dirty = b->cols;
}

void copy_in(fl_ctx* ctx, double* dst, long ldd, int n, const double* src, long lds, int p,
             int loc) {
    if (p <= 0 || n <= 0) return;
    CK(cudaMemcpy2DAsync(dst, sizeof(double) * ldd, src, sizeof(double) * lds, sizeof(double) * n,
                         p, loc == FL_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                         ctx->stream));
}

void copy_out(fl_ctx* ctx, double* dst, long ldd, int n, const double* src, long lds, int p,
              int loc) {
    if (p <= 0 || n <= 0) return;
    CK(cudaMemcpy2DAsync(dst, sizeof(double) * ldd, src, sizeof(double) * lds, sizeof(double) * n,
                         p, loc == FL_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                         ctx->stream));
}

// Host wait for the context stream. Polls an event instead of a blocking
// cudaStreamSynchronize: a blocked host thread woke up to ~100 ms late on
// the GPU boxes, stalling the launch-paced pipeline behind it (measured:
// 150 ms filter applications stretched to 250 ms at random).
void resolve_pending(fl_ctx* ctx);

void sync(fl_ctx* ctx) {
    static const bool block = std::getenv("FEASTLAB_BLOCKING_SYNC") != nullptr;
    if (block || !ctx->done) {
        CK(cudaStreamSynchronize(ctx->stream));
    } else {
        CK(cudaEventRecord(ctx->done, ctx->stream));
        cudaError_t e;
        while ((e = cudaEventQuery(ctx->done)) == cudaErrorNotReady) {
        }
        CK(e);
    }
    CK(cudaGetLastError());  // a refused launch (bad configuration) raises here
    if (!ctx->pending.empty()) resolve_pending(ctx);
}

// --------------------------------------------------------------- profiling scope
struct Prof {
    fl_ctx* ctx;
    int cls;
    double work;
    cudaStream_t st;
    cudaEvent_t a = nullptr;
    double tag = 0.0;
    Prof(fl_ctx* c, int k, double w, int launches = 1, cudaStream_t s = nullptr, double t = 0.0)
        : ctx(c), cls(k), work(w), st(s ? s : c->stream), tag(t) {
        g_launch_count += launches;
        if (ctx->prof.on) {
            a = ctx->prof.get();
            cudaEventRecord(a, st);
        }
    }
    ~Prof() {
        if (a) {
            cudaEvent_t b = ctx->prof.get();
            cudaEventRecord(b, st);
            ctx->prof.recs.push_back({cls, a, b, work, tag});
        }
    }
};

// Shape tag of a profiled GEMM-class launch (fl_ctx_profile_dump): role
// (1 trailing update, 2 in-block panel-column update, 3 in-block U12 update,
// 4 in-block U rows of a panel column, 5 solve update, 6 in-block solve
// update, 7 L_kk^-1 product, 8 solve diagonal-block product), M/64, N/64, K/16.
double shape_tag(int role, int M, int N, int K) {
    return (((double)role * 1024 + M / 64) * 1024 + N / 64) * 1024 + K / 16;
}

double* scratch(DBuf& b, size_t doubles) {
    b.ensure(sizeof(double) * std::max<size_t>(doubles, 1));
    return b.d();
}

// FEASTLAB_ZGEMM_TMA=0 keeps the cp.async kernel for the trailing updates
bool tma_updates() {
    static const bool on = [] {
        const char* e = std::getenv("FEASTLAB_ZGEMM_TMA");
        return !(e && e[0] == '0');
    }();
    return on && zgemm_mode() == 1;
}

// --------------------------------------------------------------- filter core
// Factor nodes [g0, g0+G) of the local range into factor slots [s0, s0+G).
// Look-ahead: stream `st` runs the swaps and the trailing update; stream `sp`
// factors panel k+1 as soon as its 64 columns are updated (GEMM "next"),
// concurrently with the rest of update k (GEMM "rest").
//   st: wait(P_k) laswp_k  U12_k  GEMM_next_k  rec(N_k)  GEMM_rest_k
//   sp: wait(N_{k-1})  panel_k  trinv(L_kk)  rec(P_k)
void factor_group_ldlt(fl_filter* f, int g0, int G, int s0, cudaStream_t st, cudaStream_t sp,
                       cudaEvent_t ev_panel, cudaEvent_t ev_next);

void factor_group(fl_filter* f, int g0, int G, int s0, cudaStream_t st, cudaStream_t sp,
                  cudaEvent_t ev_panel, cudaEvent_t ev_next) {
    if (f->ctx->factorization == FL_FACTOR_LDLT) {
        factor_group_ldlt(f, g0, G, s0, st, sp, ev_panel, ev_next);
        return;
    }
    fl_ctx* ctx = f->ctx;
    const int N = f->A->N, n = f->A->n;
    const long stride = (long)N * N;
    ZBatch F{f->fac_re.d() + s0 * stride, f->fac_im.d() + s0 * stride, N, stride};
    NodeShifts z{};
    for (int b = 0; b < G; ++b) {
        z.zr[b] = f->zr[f->kb + g0 + b];
        z.zi[b] = f->zi[f->kb + g0 + b];
    }
    int* ipiv = f->ipiv.i() + (long)s0 * N;
    int* ptab = f->ptab.i() + (long)s0 * (4 * FL_TILE + 1);
    int* cmap = f->cmap.i() + (long)s0 * N;
    int* btab = f->btab.i() + (long)s0 * LB_TAB;
    if (f->laswp_block) {
        Prof pr(ctx, P_LASWP, 0.0, 1, st);
        launch_perm_identity(cmap, N, G, st);
    }
    const int NB = N / FL_TILE;
    const long istride = 2L * NB * FL_TILE * FL_TILE;
    ZBatch Inv{f->inv_re.d() + s0 * istride, f->inv_im.d() + s0 * istride, FL_TILE, istride};
    {
        Prof pr(ctx, P_SHIFT, (8.0 + 16.0 * G) * N * N, 1, st);
        launch_shift(f->A->d(), N, N, F, z, G, st);
    }
    const int T = FL_TILE;
    auto E = [&](int r, int c) { return (long)c * N + r; };
    // C[r,c: +M x +nc] -= A[ar,ac: M x K] B[br,bc: K x nc]
    auto sub = [&](int M, int nc, int K, int ar, int ac, int br, int bc, int cr, int cc,
                   cudaStream_t s, int role) {
        if (M <= 0 || nc <= 0) return;
        ZGemm g{M, nc, K, F.re + E(ar, ac), F.im + E(ar, ac), N, stride,
                F.re + E(br, bc), F.im + E(br, bc), N, stride,
                F.re + E(cr, cc), F.im + E(cr, cc), N, stride};
        Prof pr(ctx, P_ZGEMM, 8.0 * M * nc * K * G, 1, s, shape_tag(role, M, nc, K));
        launch_zgemm_sub(g, G, s);
    };
    // F[k:k+64, c:c+nc] = L_kk^{-1} F[k:k+64, c:c+nc] (in place)
    auto linv = [&](int k, int c, int nc, cudaStream_t s) {
        if (nc <= 0) return;
        const long ib = (long)(k / T) * T * T;
        ZGemm u{T, nc, T, Inv.re + ib, Inv.im + ib, T, Inv.stride,
                F.re + E(k, c), F.im + E(k, c), N, stride, F.re + E(k, c), F.im + E(k, c), N,
                stride};
        Prof pr(ctx, P_TRSM, 8.0 * T * T * nc * G, 1, s, shape_tag(7, T, nc, T));
        launch_zgemm_set(u, G, s);
    };
    // one pivot table per panel of an outer block: panel j+1's must not
    // overwrite panel j's before st has applied it
    const int NPB = f->lu_panels;  // panels per outer block (2: 128 columns, 4: 256)
    int* tabs[FL_MAX_BLOCK_PANELS];
    for (int j = 0; j < NPB; ++j) tabs[j] = ptab + (long)(j * f->fac_slots) * (4 * T + 1);
    auto panel = [&](int k, int* tab) {
        Prof pr(ctx, P_PANEL, 0.0, 1, sp);  // also writes L_kk^{-1} into Inv
        launch_panel(F, N, k, ipiv, tab, Inv, G, sp, f->panel_res_rows);
    };
    auto swaps = [&](const int* tab, int a0, int a1, int b0, int b1, cudaStream_t s) {
        Prof pr(ctx, P_LASWP, 0.0, 1, s);
        launch_laswp(F, a0, a1, b0, b1, tab, G, s);
    };
    // A[c0:, cc : cc + nc] -= L[c0:, k0 : k0 + K] U[k0 : k0 + K, cc : cc + nc] by the
    // TMA-fed kernel; the sum planes of L21 and U12 are formed first (once per
    // outer block: `have_sums` for the second launch of a block)
    auto trailing = [&](int M, int nc, int K, int k0, int c0, int cc, bool have_sums) {
        if (M <= 0 || nc <= 0) return;
        const long sa = (long)N * f->sum_kb;
        if (!have_sums) {
            Prof pr(ctx, P_ZSUM, 24.0 * ((double)M * K + (double)K * (N - c0)) * G, 2, st);
            launch_zsum(F.re + E(c0, k0), F.im + E(c0, k0), N, stride, f->sum_a.d() + s0 * sa + c0, N,
                        sa, M, K, G, st);
            launch_zsum(F.re + E(k0, c0), F.im + E(k0, c0), N, stride,
                        f->sum_b.d() + s0 * sa + (long)c0 * f->sum_kb, f->sum_kb, sa, K, N - c0, G,
                        st);
        }
        ZGemmTma t{M, nc, K, c0, k0, s0, c0, 0, s0, k0, cc, s0, 0, cc, s0,
                   F.re + E(c0, cc), F.im + E(c0, cc), N, stride};
        Prof pr(ctx, P_ZGEMM, 8.0 * M * nc * K * G, 1, st, shape_tag(1, M, nc, K));
        launch_zgemm_sub_tma(f->maps, t, G, st);
    };
    // Outer blocks of NPB panels (BW = 64 NPB columns), panels k_j = k0 + 64 j.
    // The panel stream factors all of a block's panels while the main stream
    // finishes the previous block's trailing update (look-ahead); the trailing
    // update then has K = BW (C-tile traffic and GEMM fill/drain per flop fall
    // as 1/BW):
    //   sp: for j: [ panel j-1's swaps on the block's columns left of it |
    //               panels 0..j-1's swaps on panel j's columns |
    //               U rows k_0..k_j of panel j's columns (L_ii^-1 and in-block
    //               updates) | A[k_j:, panel j] -= L[k_j:, k_0:k_j] U ] panel j
    //                                                                -> ev_panel
    //   st: every panel's swaps on the other columns | the block's U rows of
    //       the columns right of it (L_jj^-1, in-block updates) |
    //       A[c0:, c0:] -= L[c0:, block] U[block, c0:]  (the next block's BW
    //       columns first -> ev_next, then the remainder)
    CK(cudaEventRecord(ev_next, st));  // shift done: block 0 may start
    for (int k0 = 0; k0 < N; k0 += NPB * T) {
        const int np = std::min(NPB, (N - k0) / T);
        const int c0 = k0 + np * T;
        CK(cudaStreamWaitEvent(sp, ev_next, 0));
        for (int j = 0; j < np; ++j) {
            const int kj = k0 + j * T;
            if (j > 0) {
                // the block's earlier L columns must carry panel j-1's
                // interchanges before they update panel j (the last panel's
                // reach them on st, off the look-ahead chain)
                if (!f->laswp_block) {
                    if (j >= 2) swaps(tabs[j - 1], k0, kj - T, 0, 0, sp);
                    for (int i = 0; i < j; ++i) swaps(tabs[i], kj, kj + T, 0, 0, sp);
                }
                for (int i = 0; i < j; ++i) {
                    const int ki = k0 + i * T;
                    linv(ki, kj, T, sp);
                    if (i + 1 < j) sub((j - 1 - i) * T, T, T, ki + T, ki, ki, kj, ki + T, kj, sp, 4);
                }
                sub(N - kj, T, j * T, kj, k0, k0, kj, kj, kj, sp, 2);
            }
            panel(kj, tabs[j]);
            // one pass per panel over the block's other columns (the last
            // panel's reach the columns left of it on st)
            if (f->laswp_block && j + 1 < np) swaps(tabs[j], k0, kj, kj + T, c0, sp);
        }
        CK(cudaEventRecord(ev_panel, sp));
        CK(cudaStreamWaitEvent(st, ev_panel, 0));
        const int rest = N - c0;
        if (f->laswp_block && np >= 2) {
            // the columns outside the block take the composition of the block's
            // np net permutations in one pass; the block's own columns left of
            // its last panel still lack that panel's interchanges
            {
                Prof pr(ctx, P_LASWP, 0.0, 2, st);
                launch_laswp_block(F, N, k0, np, 0, k0, c0, N, tabs[0],
                                   (long)f->fac_slots * (4 * T + 1), cmap, btab, G, st);
            }
            swaps(tabs[np - 1], k0, k0 + (np - 1) * T, 0, 0, st);
        } else {
            for (int j = 0; j < np; ++j) {
                // panels 1..np-2 already swapped the block's columns left of them (sp)
                const int left = j == np - 1 ? k0 + j * T : k0;
                if (rest > 0) swaps(tabs[j], 0, left, c0, N, st);
                else swaps(tabs[j], 0, left, 0, 0, st);
            }
        }
        if (rest <= 0) break;
        for (int j = 0; j < np; ++j) {
            const int kj = k0 + j * T;
            linv(kj, c0, rest, st);
            if (j + 1 < np) sub((np - 1 - j) * T, rest, T, kj + T, kj, kj, c0, kj + T, c0, st, 3);
        }
        const int nxt = std::min(np * T, rest);
        if (f->maps_ok && tma_updates() && np * T >= 2 * T && np * T <= f->sum_kb) {
            trailing(rest, nxt, np * T, k0, c0, c0, false);
            CK(cudaEventRecord(ev_next, st));
            trailing(rest, rest - nxt, np * T, k0, c0, c0 + nxt, true);
        } else {
            sub(rest, nxt, np * T, c0, k0, k0, c0, c0, c0, st, 1);
            CK(cudaEventRecord(ev_next, st));
            sub(rest, rest - nxt, np * T, c0, k0, k0, c0 + nxt, c0, c0 + nxt, st, 1);
        }
    }
    Prof pr(ctx, P_PANEL, 0.0, 3, st);
    launch_trinv(F, 0, NB, true, Inv, NB, G, st);  // U_ii^{-1} for the solves
    launch_check_diag(F, n, G, f->kb + g0, f->bad.i(), st);  // global node index
    launch_ipiv_to_perm(ipiv, f->perm.i() + (long)s0 * N, N, G, st);
}

// Complex-symmetric LDL^T (FL_FACTOR_LDLT, ldlt.cu) of nodes [g0, g0+G) into
// factor slots [s0, ...): same factor layout as factor_group (L, U = D L^T,
// identity permutation), trailing updates on the lower trapezoid only.
// Outer blocks of NPB panels with the LU's look-ahead split:
//   sp: for panel j of the block: A[k_j:, panel j] -= L[k_j:, k_0:k_j] U[k_0:k_j, panel j]
//       | ldlt_panel | W = A[k_j+64:, panel j] L_jj^{-T} | split (L = W D^{-1}, U = W^T)
//                                                                      -> ev_panel
//   st: A[c0:, c0:] -= L[c0:, block] U[block, c0:], lower tiles: the next
//       block's columns first -> ev_next, then the remainder
// The remainder of block b-1 (rows and columns >= c0 of block b... lower
// tiles) never touches the rows [k0, c0) or columns [k0, c0) block b's panel
// chain writes, so the two streams need no other ordering.
void factor_group_ldlt(fl_filter* f, int g0, int G, int s0, cudaStream_t st, cudaStream_t sp,
                       cudaEvent_t ev_panel, cudaEvent_t ev_next) {
    fl_ctx* ctx = f->ctx;
    const int N = f->A->N, n = f->A->n;
    const long stride = (long)N * N;
    ZBatch F{f->fac_re.d() + s0 * stride, f->fac_im.d() + s0 * stride, N, stride};
    NodeShifts z{};
    for (int b = 0; b < G; ++b) {
        z.zr[b] = f->zr[f->kb + g0 + b];
        z.zi[b] = f->zi[f->kb + g0 + b];
    }
    const int NB = N / FL_TILE;
    const long istride = 2L * NB * FL_TILE * FL_TILE;
    ZBatch Inv{f->inv_re.d() + s0 * istride, f->inv_im.d() + s0 * istride, FL_TILE, istride};
    const int T = FL_TILE;
    const long lts = (long)T * T;
    double* ltr = f->lt_re.d() + s0 * lts;
    double* lti = f->lt_im.d() + s0 * lts;
    {
        Prof pr(ctx, P_SHIFT, (8.0 + 16.0 * G) * N * N, 1, st);
        launch_shift(f->A->d(), N, N, F, z, G, st);
    }
    auto E = [&](int r, int c) { return (long)c * N + r; };
    // C[cr, cc: M x nc] -= A[ar, ac: M x K] B[br, bc: K x nc]; lower >= 0: only
    // the tiles on or below the global diagonal (tri_s = (cc - cr) / 64)
    auto sub = [&](int M, int nc, int K, int ar, int ac, int br, int bc, int cr, int cc,
                   cudaStream_t s, bool lower) {
        if (M <= 0 || nc <= 0) return;
        ZGemm g{M, nc, K, F.re + E(ar, ac), F.im + E(ar, ac), N, stride,
                F.re + E(br, bc), F.im + E(br, bc), N, stride,
                F.re + E(cr, cc), F.im + E(cr, cc), N, stride};
        const int ts = (cc - cr) / T;
        // algorithmic work: the tiles computed
        double tiles = 0;
        if (lower) {
            for (int c = 0; c < nc / T; ++c) {
                const int lo = std::max(0, c + ts);
                if (lo < M / T) tiles += M / T - lo;
            }
        } else {
            tiles = (double)(M / T) * (nc / T);
        }
        Prof pr(ctx, P_ZGEMM, 8.0 * tiles * T * T * K * G, 1, s);
        if (lower) launch_zgemm_sub_lower(g, ts, G, s);
        else launch_zgemm_sub(g, G, s);
    };
    // the lower-trapezoid trailing update by the TMA-fed kernel (cf. factor_group)
    auto trailing = [&](int M, int nc, int K, int k0, int c0, int cc, bool have_sums) {
        if (M <= 0 || nc <= 0) return;
        const long sa = (long)N * f->sum_kb;
        if (!have_sums) {
            Prof pr(ctx, P_ZSUM, 24.0 * ((double)M * K + (double)K * (N - c0)) * G, 2, st);
            launch_zsum(F.re + E(c0, k0), F.im + E(c0, k0), N, stride, f->sum_a.d() + s0 * sa + c0, N,
                        sa, M, K, G, st);
            launch_zsum(F.re + E(k0, c0), F.im + E(k0, c0), N, stride,
                        f->sum_b.d() + s0 * sa + (long)c0 * f->sum_kb, f->sum_kb, sa, K, N - c0, G,
                        st);
        }
        ZGemmTma t{M, nc, K, c0, k0, s0, c0, 0, s0, k0, cc, s0, 0, cc, s0,
                   F.re + E(c0, cc), F.im + E(c0, cc), N, stride};
        t.tri = true;
        t.tri_s = (cc - c0) / T;
        double tiles = 0;
        for (int c = 0; c < nc / T; ++c) {
            const int lo = std::max(0, c + t.tri_s);
            if (lo < M / T) tiles += M / T - lo;
        }
        Prof pr(ctx, P_ZGEMM, 8.0 * tiles * T * T * K * G, 1, st, shape_tag(1, M, nc, K));
        launch_zgemm_sub_tma(f->maps, t, G, st);
    };
    const int NPB = f->lu_panels;
    CK(cudaEventRecord(ev_next, st));  // shift done: block 0 may start
    for (int k0 = 0; k0 < N; k0 += NPB * T) {
        const int np = std::min(NPB, (N - k0) / T);
        const int c0 = k0 + np * T;
        CK(cudaStreamWaitEvent(sp, ev_next, 0));
        for (int j = 0; j < np; ++j) {
            const int kj = k0 + j * T;
            if (j > 0) sub(N - kj, T, j * T, kj, k0, k0, kj, kj, kj, sp, true);
            {
                Prof pr(ctx, P_PANEL, 0.0, 1, sp);
                launch_ldlt_panel(F, kj, Inv, ltr, lti, lts, G, sp);
            }
            const int rows = N - kj - T;
            if (rows > 0) {
                ZGemm w{rows, T, T, F.re + E(kj + T, kj), F.im + E(kj + T, kj), N, stride,
                        ltr, lti, T, lts, F.re + E(kj + T, kj), F.im + E(kj + T, kj), N, stride};
                {
                    Prof pr(ctx, P_TRSM, 8.0 * rows * T * T * G, 1, sp);
                    launch_zgemm_set(w, G, sp);
                }
                Prof pr(ctx, P_LASWP, 0.0, 1, sp);  // the split's data movement
                launch_ldlt_split(F, kj, kj + T, rows, G, sp);
            }
        }
        CK(cudaEventRecord(ev_panel, sp));
        CK(cudaStreamWaitEvent(st, ev_panel, 0));
        const int rest = N - c0;
        if (rest <= 0) break;
        const int nxt = std::min(np * T, rest);
        if (f->maps_ok && tma_updates() && np * T >= 2 * T && np * T <= f->sum_kb) {
            trailing(rest, nxt, np * T, k0, c0, c0, false);
            CK(cudaEventRecord(ev_next, st));
            trailing(rest, rest - nxt, np * T, k0, c0, c0 + nxt, true);
        } else {
            sub(rest, nxt, np * T, c0, k0, k0, c0, c0, c0, st, true);
            CK(cudaEventRecord(ev_next, st));
            sub(rest, rest - nxt, np * T, c0, k0, k0, c0 + nxt, c0, c0 + nxt, st, true);
        }
    }
    Prof pr(ctx, P_PANEL, 0.0, 3, st);
    launch_trinv(F, 0, NB, true, Inv, NB, G, st);  // U_ii^{-1} for the solves
    launch_check_diag(F, n, G, f->kb + g0, f->bad.i(), st);
    launch_iota_perm(f->perm.i() + (long)s0 * N, N, G, st);
}

// W_b = (z_b I - A)^{-1} X for nodes [g0, g0+G) using factor slots [s0, ...).
void solve_group(fl_filter* f, int g0, int G, int s0, const double* X, long ldx, int P,
                 cudaStream_t st) {
    fl_ctx* ctx = f->ctx;
    const int N = f->A->N;
    const long stride = (long)N * N;
    ZBatch F{f->fac_re.d() + s0 * stride, f->fac_im.d() + s0 * stride, N, stride};
    ZBatch W{f->w_re.d() + g0 * f->w_stride, f->w_im.d() + g0 * f->w_stride, N, f->w_stride};
    {
        Prof pr(ctx, P_PERMUTE, 24.0 * N * P * G, 1, st);
        launch_permute_rhs(X, ldx, N, P, f->perm.i() + (long)s0 * N, W, G, st);
    }
    const int NB = N / FL_TILE;
    const long istride = 2L * NB * FL_TILE * FL_TILE;
    ZBatch Inv{f->inv_re.d() + s0 * istride, f->inv_im.d() + s0 * istride, FL_TILE, istride};
    auto tri = [&](int blk, int r0) {  // W_i <- T_ii^{-1} W_i (DMMA, in place)
        Prof pr(ctx, P_TRSM, 8.0 * FL_TILE * FL_TILE * P * G, 1, st,
                shape_tag(8, FL_TILE, P, FL_TILE));
        ZGemm u{FL_TILE, P, FL_TILE,
                Inv.re + (long)blk * FL_TILE * FL_TILE, Inv.im + (long)blk * FL_TILE * FL_TILE,
                FL_TILE, Inv.stride,
                W.re + r0, W.im + r0, N, W.stride, W.re + r0, W.im + r0, N, W.stride};
        launch_zgemm_set(u, G, st);
    };
    // W[wr: +M] -= F[fr: +M, fc: +K] W[wk: +K]
    auto sub = [&](int M, int K, int fr, int fc, int wk, int wr) {
        if (M <= 0) return;
        ZGemm g{M, P, K, F.re + (long)fc * N + fr, F.im + (long)fc * N + fr, N, stride,
                W.re + wk, W.im + wk, N, W.stride, W.re + wr, W.im + wr, N, W.stride};
        Prof pr(ctx, P_ZGEMM, 8.0 * M * P * K * G, 1, st, shape_tag(K > FL_TILE ? 5 : 6, M, P, K));
        launch_zgemm_sub(g, G, st);
    };
    // row blocks of NPB tiles (cf. the LU), so the long updates have K = 64 NPB:
    // forward (unit lower), block [r0, r0 + np 64): W_j = L_jj^-1 W_j and the
    //   in-block updates below it, then W[r0 + np 64:] -= L[.., block] W_block
    const int T = FL_TILE;
    const int NPB = f->solve_panels;
    for (int ib = 0; ib < NB; ib += NPB) {
        const int np = std::min(NPB, NB - ib), r0 = ib * T;
        for (int j = 0; j < np; ++j) {
            const int rj = r0 + j * T;
            tri(ib + j, rj);
            if (j + 1 < np) sub((np - 1 - j) * T, T, rj + T, rj, rj, rj + T);
        }
        sub(N - r0 - np * T, np * T, r0 + np * T, r0, r0, r0 + np * T);
    }
    // backward (upper), blocks aligned to the end: within a block from its
    // last tile up (W_j = U_jj^-1 W_j, then the in-block rows above it), then
    // W[:r0] -= U[:r0, block] W_block
    for (int ie = NB; ie > 0; ie -= NPB) {
        const int np = std::min(NPB, ie), ib = ie - np, r0 = ib * T;
        for (int j = np - 1; j >= 0; --j) {
            const int rj = r0 + j * T;
            tri(NB + ib + j, rj);
            if (j > 0) sub(j * T, T, r0, rj, rj, r0);
        }
        sub(r0, np * T, 0, r0, r0, 0);
    }
}

// FEASTLAB_GRAPHS=0 disables the CUDA-graph replay of filter applications
bool graphs_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("FEASTLAB_GRAPHS");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Few local nodes (latency-bound: the per-node LU chain sets the step time,
// e.g. 2 nodes per GPU at 8 GPUs) -> the on-chip panel for every panel of
// <= 4096 rows; many local nodes (throughput-bound: panels overlap other
// chunks' GEMMs) -> the on-chip panel only below FEASTLAB_PANEL_RES_ROWS rows
// (default 2048), so tall panels keep co-residing with GEMM CTAs.
int panel_res_rows(int local_nodes) {
    static const int thr = [] {
        const char* e = std::getenv("FEASTLAB_PANEL_RES_ROWS");
        return e ? std::atoi(e) : 2048;
    }();
    static const int few = [] {
        const char* e = std::getenv("FEASTLAB_PANEL_FEW_NODES");
        return e ? std::atoi(e) : 4;
    }();
    return local_nodes <= few ? 4096 : thr;
}

// Panels per LU outer block (1..16) / tiles per triangular-solve row block (1..8).
// Many local nodes (throughput-bound): 4 (16 when N >= 12288; 8 for fewer nodes there), so the trailing
// updates run with K = 256 (1024; cfg4 LU 11.36 -> 11.21 s, LDL^T 5.48 -> 5.39 s
// against 8 panels); few (latency-bound: the per-node panel chain sets the step time):
// 2, so the look-ahead stream has half as many panels to factor per block.
int block_panels(const char* env, int dflt, int most) {
    const char* e = std::getenv(env);
    const int v = e ? std::atoi(e) : dflt;
    return std::max(1, std::min(most, v));
}

// Serialises the free-memory read and the allocation of factor slots per
// device: concurrent solves on one GPU (solve_concurrently, per_device > 1)
// each see the memory the others already took.
std::mutex& device_alloc_mutex(int device) {
    static std::mutex mu[64];
    return mu[device & 63];
}

size_t free_bytes() {
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    return fr;
}

// X, Y: device, N x P padded (zero rows >= n, zero cols >= p); P multiple of 64.
void filter_apply_dev(fl_filter* f, const double* X, long ldx, int p, double* Y, long ldy,
                      long long* rhs, long long* facts) {
    fl_ctx* ctx = f->ctx;
    const int N = f->A->N;
    const int P = round_up(p, FL_TILE);
    const int L = f->ke - f->kb;
    const long fstride = (long)N * N;
    // W for every local node
    if (f->w_P < P || f->w_stride != (long)N * P) {
        f->w_stride = (long)N * P;
        f->w_re.ensure(sizeof(double) * (size_t)f->w_stride * std::max(L, 1));
        f->w_im.ensure(sizeof(double) * (size_t)f->w_stride * std::max(L, 1));
        f->w_P = P;
    }
    // factor slots
    std::unique_lock<std::mutex> alloc_lk(device_alloc_mutex(ctx->device));
    int slots;
    if (f->cache) {
        slots = L;
    } else {
        const size_t per = sizeof(double) * 2 * (size_t)fstride + sizeof(int) * 2 * (size_t)N;
        const size_t budget = (size_t)(0.6 * (double)(free_bytes() + f->fac_re.bytes + f->fac_im.bytes));
        slots = (int)std::max<size_t>(1, std::min<size_t>((size_t)L, budget / per));
        slots = std::min(slots, 16);
    }
    if (f->fac_slots < slots) {
        f->fac_re.release();
        f->fac_im.release();
        f->fac_re.ensure(sizeof(double) * (size_t)fstride * slots);
        f->fac_im.ensure(sizeof(double) * (size_t)fstride * slots);
        f->ipiv.ensure(sizeof(int) * (size_t)N * slots);
        f->perm.ensure(sizeof(int) * (size_t)N * slots);
        f->ptab.ensure(sizeof(int) * (size_t)(4 * FL_TILE + 1) * FL_MAX_BLOCK_PANELS * slots);
        f->cmap.ensure(sizeof(int) * (size_t)N * slots);
        f->btab.ensure(sizeof(int) * (size_t)LB_TAB * slots);
        f->inv_re.ensure(sizeof(double) * 2 * (size_t)N * FL_TILE * slots);
        f->inv_im.ensure(sizeof(double) * 2 * (size_t)N * FL_TILE * slots);
        f->lt_re.ensure(sizeof(double) * (size_t)FL_TILE * FL_TILE * slots);
        f->lt_im.ensure(sizeof(double) * (size_t)FL_TILE * FL_TILE * slots);
        f->fac_slots = slots;
        f->maps_ok = false;
        std::fill(f->factored.begin(), f->factored.end(), 0);
    }
    alloc_lk.unlock();
    if (f->fac_mode != ctx->factorization) {  // cached factors of the other kind
        std::fill(f->factored.begin(), f->factored.end(), 0);
        f->fac_mode = ctx->factorization;
    }
    f->bad.ensure(sizeof(int) * 4);
    if (!f->h_bad) CK(cudaMallocHost(&f->h_bad, sizeof(int) * 4));
    // Node chunks run concurrently on the context's auxiliary streams so one
    // chunk's latency-bound panels overlap another chunk's DMMA GEMMs.
    const int ns = std::max(1, std::min(std::min(L, slots), ctx->nstreams));
    f->panel_res_rows = panel_res_rows(L);
    // wide outer blocks (16 panels: K = 1024 trailing updates) pay off only on
    // large matrices (cfg4: -3 % against 4 panels; cfg2 / cfg3: +5 % / +3 %,
    // the longer in-block chain); at n >= 12288 even 4 local nodes take 8
    // (cfg4 8-GPU shard 1530 -> 1467 ms against 2 panels)
    f->lu_panels = block_panels("FEASTLAB_LU_PANELS",
                                 N >= 12288 ? (L >= 8 ? 16 : 8) : (L >= 8 ? 4 : 2),
                                 FL_MAX_BLOCK_PANELS);
    f->solve_panels = block_panels("FEASTLAB_SOLVE_PANELS", 4, 8);
    {
        const char* e = std::getenv("FEASTLAB_LASWP_BLOCK");
        f->laswp_block = !(e && e[0] == '0');
    }
    // sum planes and tensor maps of the TMA-fed trailing updates (outer blocks
    // of at least 128 columns, 3M product)
    if (tma_updates() && f->lu_panels >= 2 &&
        (!f->maps_ok || f->sum_kb != f->lu_panels * FL_TILE ||
         f->sum_a.bytes < sizeof(double) * (size_t)N * f->lu_panels * FL_TILE * f->fac_slots)) {
        const int KB = f->lu_panels * FL_TILE;
        f->sum_a.ensure(sizeof(double) * (size_t)N * KB * f->fac_slots);
        f->sum_b.ensure(sizeof(double) * (size_t)N * KB * f->fac_slots);
        f->sum_kb = KB;
        make_tma_map_mk(&f->maps.Ar, f->fac_re.d(), N, N, N, fstride, f->fac_slots);
        make_tma_map_mk(&f->maps.Ai, f->fac_im.d(), N, N, N, fstride, f->fac_slots);
        make_tma_map_mk(&f->maps.As, f->sum_a.d(), N, KB, N, (long)N * KB, f->fac_slots);
        make_tma_map_km(&f->maps.Br, f->fac_re.d(), N, N, N, fstride, f->fac_slots);
        make_tma_map_km(&f->maps.Bi, f->fac_im.d(), N, N, N, fstride, f->fac_slots);
        make_tma_map_km(&f->maps.Bs, f->sum_b.d(), KB, N, KB, (long)KB * N, f->fac_slots);
        f->maps_ok = true;
    }
    long long new_facts = 0;
    // everything below is stream work only (no host synchronisation), so a
    // non-cache application is one CUDA graph: ~2.8k launches on 9 streams
    // replayed with one cudaGraphLaunch instead of host-paced launches
    bool needs_factor = !f->cache;
    if (f->cache)
        for (char d : f->factored) needs_factor |= !d;
    auto enqueue = [&] {
        // sentinel 0x7f7f7f7f = no singular node. Only an application that
        // factors resets it: a solve-only application (cached factors) keeps
        // the verdict of the application that built them, so a singular node
        // is raised even when the caller applies again before syncing
        if (needs_factor) CK(cudaMemsetAsync(f->bad.p, 0x7f, sizeof(int), ctx->stream));
        CK(cudaEventRecord(ctx->fork, ctx->stream));
        for (int j = 0; j < ns; ++j) CK(cudaStreamWaitEvent(ctx->aux[j], ctx->fork, 0));
        if (f->cache) {
            // chunk j = nodes [j*L/ns, (j+1)*L/ns); factor the uncached ones, then solve
            for (int j = 0; j < ns; ++j) {
                const int c0 = (int)((long)L * j / ns), c1 = (int)((long)L * (j + 1) / ns);
                int g = c0;
                while (g < c1) {
                    if (f->factored[g]) { ++g; continue; }
                    int e = g;  // a run of unfactored nodes, at most 16 per batch
                    while (e < c1 && e - g < 16 && !f->factored[e]) ++e;
                    factor_group(f, g, e - g, g, ctx->aux[j], ctx->paux[j], ctx->ev_panel[j],
                                 ctx->ev_next[j]);
                    for (int k = g; k < e; ++k) f->factored[k] = 1;
                    new_facts += e - g;
                    g = e;
                }
                if (c1 > c0) solve_group(f, c0, c1 - c0, c0, X, ldx, P, ctx->aux[j]);
            }
        } else {
            // rounds of `slots` nodes; round chunk j reuses slots [j*slots/ns, ...) on stream j
            for (int g = 0; g < L; g += slots) {
                const int G = std::min(slots, L - g);
                const int nsr = std::min(ns, G);
                for (int j = 0; j < nsr; ++j) {
                    const int c0 = (int)((long)G * j / nsr), c1 = (int)((long)G * (j + 1) / nsr);
                    const int s0 = (int)((long)slots * j / ns);
                    factor_group(f, g + c0, c1 - c0, s0, ctx->aux[j], ctx->paux[j],
                                 ctx->ev_panel[j], ctx->ev_next[j]);
                    solve_group(f, g + c0, c1 - c0, s0, X, ldx, P, ctx->aux[j]);
                }
            }
            new_facts = f->nc;
        }
        for (int j = 0; j < ns; ++j) {
            CK(cudaEventRecord(ctx->join[j], ctx->aux[j]));
            CK(cudaStreamWaitEvent(ctx->stream, ctx->join[j], 0));
        }
        // ordered accumulation over the local nodes, in launches of at most
        // kMaxNodes weights (a later launch continues the same ascending sum
        // from Y: the association is unchanged)
        auto weights = [&](int b0, int cnt) {
            NodeShifts w{};
            for (int b = 0; b < cnt; ++b) {
                w.zr[b] = f->wr[f->kb + b0 + b];
                w.zi[b] = f->wi[f->kb + b0 + b];
            }
            return w;
        };
        ZBatch W{f->w_re.d(), f->w_im.d(), N, f->w_stride};
        auto wslice = [&](int b0) {
            return ZBatch{W.re + b0 * W.stride, W.im + b0 * W.stride, W.ld, W.stride};
        };
        if (ctx->comm && ctx->reduction == FL_REDUCE_ORDERED) {
            // every rank's terms at slot rank * Lmax + local index; all-gather;
            // ascending global-k sum on every rank (bitwise G-invariant)
            if (ldy != N) throw Fail{FL_INVALID_ARGUMENT, "ordered reduction needs a packed Y"};
            const int G = ctx->nranks;
            const int Lmax = (f->nc + G - 1) / G;
            const long ts = (long)N * P;
            double* T = scratch(f->terms, (size_t)std::max(Lmax, 1) * ts);
            double* Tall = scratch(f->terms_all, (size_t)G * std::max(Lmax, 1) * ts);
            std::vector<int> slot(f->nc);
            for (int r = 0; r < G; ++r) {
                int b0 = 0, b1 = 0;
                fl_node_shard(f->nc, r, G, &b0, &b1);
                for (int k = b0; k < b1; ++k) slot[k] = r * Lmax + (k - b0);
            }
            for (int b0 = 0; b0 < L; b0 += kMaxNodes) {
                const int cnt = std::min(kMaxNodes, L - b0);
                Prof pr(ctx, P_ACCUM, 24.0 * cnt * N * P);
                launch_node_terms(wslice(b0), N, P, weights(b0, cnt), cnt, T + b0 * ts, ts,
                                  ctx->stream);
            }
            Prof pr(ctx, P_ALLREDUCE, 8.0 * G * Lmax * ts, 1);
            nccl_check(ncclAllGather(T, Tall, (size_t)Lmax * ts, ncclFloat64, ctx->comm,
                                     ctx->stream),
                       "ncclAllGather(node terms)");
            for (int k0 = 0; k0 < f->nc; k0 += kMaxNodes) {
                NodeSlots sl{};
                const int cnt = std::min(kMaxNodes, f->nc - k0);
                for (int k = 0; k < cnt; ++k) sl.slot[k] = slot[k0 + k];
                launch_ordered_sum(Tall, ts, sl, cnt, N, P, Y, ldy, k0 > 0, ctx->stream);
            }
            nccl_check(ncclAllReduce(f->bad.p, f->bad.p, 1, ncclInt32, ncclMin, ctx->comm,
                                     ctx->stream),
                       "ncclAllReduce(bad node)");
        } else if (L > 0) {
            for (int b0 = 0; b0 < L; b0 += kMaxNodes) {
                const int cnt = std::min(kMaxNodes, L - b0);
                Prof pr(ctx, P_ACCUM, (16.0 * cnt + (b0 > 0 ? 16.0 : 8.0)) * N * P);
                launch_accumulate(wslice(b0), N, P, weights(b0, cnt), cnt, Y, ldy, b0 > 0,
                                  ctx->stream);
            }
        } else {
            CK(cudaMemsetAsync(Y, 0, sizeof(double) * (size_t)ldy * P, ctx->stream));
        }
        if (ctx->comm && ctx->reduction != FL_REDUCE_ORDERED) {
            if (ldy != N) throw Fail{FL_INVALID_ARGUMENT, "allreduce needs a packed Y"};
            Prof pr(ctx, P_ALLREDUCE, 8.0 * N * p, 0);
            nccl_check(ncclAllReduce(Y, Y, (size_t)N * p, ncclFloat64, ncclSum, ctx->comm,
                                     ctx->stream),
                       "ncclAllReduce(Y)");
            // every rank learns the first singular node, so all of them throw
            nccl_check(ncclAllReduce(f->bad.p, f->bad.p, 1, ncclInt32, ncclMin, ctx->comm,
                                     ctx->stream),
                       "ncclAllReduce(bad node)");
        }
    };
    // Graph policy: an application is pure stream work, so it is captured and
    // replayed while its launch key holds. Eager (host-paced) launches enqueue
    // chunk after chunk, and once a stream's launch queue is full the host
    // blocks on it while the other chunks' streams wait for work: cfg4's LU
    // (54k launches) runs 13.3 s eagerly against 11.4 s as one graph, while
    // capture + instantiate cost 0.4 s. So large problems (N >= 2048) capture
    // on the first call; small ones on the second (their capture costs more
    // than an eager application saves). Cached factorizations: the factoring
    // application is captured too (launched once, phase 1), the solve-only
    // ones are replayed (phase 2).
    const int phase = f->cache ? (needs_factor ? 1 : 2) : 0;
    const fl_filter::GraphKey key{X, Y, f->fac_re.p, f->w_re.p, ldx, ldy, p, slots, ns,
                                  zgemm_mode(), ctx->reduction, ctx->factorization, phase,
                                  f->lu_panels, f->solve_panels, f->panel_res_rows,
                                  f->laswp_block};
    const bool graphable = !ctx->prof.on && graphs_enabled();
    const bool big = N >= 2048;
    if (graphable && f->gexec && f->gkey == key && phase != 1) {
        CK(cudaGraphLaunch(f->gexec, ctx->stream));
        g_launch_count += f->glaunches;
        new_facts = f->cache ? 0 : f->nc;
    } else if (graphable && (f->gseen == key || big)) {
        if (f->gexec) {  // an in-flight launch of it completes first
            cudaGraphExecDestroy(f->gexec);
            f->gexec = nullptr;
        }
        const std::vector<char> factored0 = f->factored;
        const long long l0 = g_launch_count;
        CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed));
        cudaGraph_t graph = nullptr;
        try {
            enqueue();
            launch_check(cudaGetLastError(), "filter application (capture)");
        } catch (...) {
            cudaStreamEndCapture(ctx->stream, &graph);
            if (graph) cudaGraphDestroy(graph);
            f->factored = factored0;
            throw;
        }
        CK(cudaStreamEndCapture(ctx->stream, &graph));
        // keep the look-ahead panel stream's priority on its captured kernel nodes
        const cudaError_t e =
            cudaGraphInstantiate(&f->gexec, graph, cudaGraphInstantiateFlagUseNodePriority);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) f->factored = factored0;
        CK(e);
        f->glaunches = g_launch_count - l0;
        f->gkey = key;
        f->gseen = key;
        CK(cudaGraphLaunch(f->gexec, ctx->stream));
    } else {
        f->gseen = key;
        enqueue();
        launch_check(cudaGetLastError(), "filter application");
    }
    // the singular-node verdict travels to pinned memory behind the work; the
    // host does not wait for it here (a host round trip per application
    // exposed host scheduling jitter to the GPU timeline): the next sync() on
    // the context -- every host-returning call makes one -- raises it
    CK(cudaMemcpyAsync(f->h_bad, f->bad.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    if (!f->check_pending) {
        f->check_pending = true;
        ctx->pending.push_back(f);
    }
    if (f->cache && ctx->comm) {
        // factorizations are counted globally: every rank adds the same total
        long long loc = new_facts, tot = 0;
        DBuf t;
        t.ensure(sizeof(long long));
        CK(cudaMemcpyAsync(t.p, &loc, sizeof(long long), cudaMemcpyHostToDevice, ctx->stream));
        nccl_check(ncclAllReduce(t.p, t.p, 1, ncclInt64, ncclSum, ctx->comm, ctx->stream),
                   "ncclAllReduce(facts)");
        CK(cudaMemcpyAsync(&tot, t.p, sizeof(long long), cudaMemcpyDeviceToHost, ctx->stream));
        sync(ctx);
        new_facts = tot;
    }
    if (rhs) *rhs += (long long)f->nc * p;
    if (facts) *facts += new_facts;
}

// Raise the first singular node among the applications whose verdicts have
// arrived (called by sync() after the stream drained).
void resolve_pending(fl_ctx* ctx) {
    fl_filter* bad = nullptr;
    for (fl_filter* f : ctx->pending) {
        f->check_pending = false;
        if (!bad && *f->h_bad != 0x7f7f7f7f) bad = f;
    }
    ctx->pending.clear();
    if (!bad) return;
    const int k = *bad->h_bad;
    if (bad->cache) std::fill(bad->factored.begin(), bad->factored.end(), 0);
    char buf[256];
    std::snprintf(buf, sizeof(buf), "factorize_node: singular factorization at node %d (z = %f+%fi)",
                  k, bad->zr[k], bad->zi[k]);
    Fail fl{FL_SINGULAR_NODE, buf};
    fl.index = k;
    fl.zr = bad->zr[k];
    fl.zi = bad->zi[k];
    throw fl;
}

// --------------------------------------------------------------- Rayleigh-Ritz helpers

// Symmetric eigensolve of the p x p matrix M (device, ld ldm, destroyed):
// ascending vals (device), vectors into V (P x P zero-padded, ld P).
void device_sym_eig(fl_ctx* ctx, double* M, long ldm, int p, int P, double* vals, double* V,
                    double* work, double* Vtmp) {
    Prof pr(ctx, P_EIG, (double)p, 0);
    launch_fro2(M, ldm, p, ctx->scal.d(), ctx->stream);
    double fro2 = 0.0;
    CK(cudaMemcpyAsync(&fro2, ctx->scal.p, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    static const bool scalar = [] {
        const char* e = std::getenv("FEASTLAB_EIG");
        return e && std::strcmp(e, "scalar") == 0;
    }();
    if (!scalar) {
        // block Jacobi (ritz.cu); the output V doubles as its Q-block buffer
        int sweeps = 0;
        const int rc = block_jacobi_eig(M, ldm, p, P, std::sqrt(fro2), work, Vtmp, V, vals, V, P,
                                        reinterpret_cast<unsigned long long*>(ctx->cnt.p),
                                        ctx->h_cnt, 40, &sweeps, ctx->stream);
        g_launch_count += 2 + 2LL * sweeps * (P / 32 - 1);
        static const bool dbg = std::getenv("FEASTLAB_EIG_DEBUG") != nullptr;
        if (dbg) std::fprintf(stderr, "block_jacobi_eig: p=%d sweeps=%d\n", p, sweeps);
        if (rc != 0) throw Fail{FL_CUDA, "block_jacobi_eig failed"};
        CK(cudaGetLastError());
        return;
    }
    CK(cudaMemsetAsync(V, 0, sizeof(double) * (size_t)P * P, ctx->stream));
    CK(cudaMemsetAsync(Vtmp, 0, sizeof(double) * (size_t)P * P, ctx->stream));
    const int rc = jacobi_eig(M, ldm, p, std::sqrt(fro2), work, Vtmp, P, vals, V, P,
                              ctx->ints.i(), reinterpret_cast<unsigned long long*>(ctx->cnt.p), 40,
                              ctx->stream);
    g_launch_count += 4;
    if (rc != 0) throw Fail{FL_CUDA, "jacobi_eig: cooperative launch failed"};
    CK(cudaGetLastError());
}

void ensure_rr_scratch(fl_ctx* ctx) {
    ctx->chol_info.ensure(64);
    ctx->ints.ensure(64);
    ctx->cnt.ensure(sizeof(unsigned long long) * 64);
    ctx->scal.ensure(64);
}

// ColPivHouseholderQR(X) with threshold thr (proj/src/ritz.cpp:22-29,
// drivers.cpp:33-36): rank = #{|R_kk| > thr * max |R_jj|}; if U is given it
// receives the first `rank` columns of Q.
int colpiv_qr(fl_ctx* ctx, const fl_block* X, double thr, fl_block* U) {
    const int n = X->n, N = X->N, p = X->cols;
    const int kmax = std::min(n, p);
    double* Aw = scratch(ctx->rr_nxp, (size_t)N * std::max(p, 1));
    double* tau = scratch(ctx->vals_d, std::max(kmax, 1));
    double* vn = scratch(ctx->norms_d, 2 * (size_t)std::max(p, 1));
    int* jpvt = reinterpret_cast<int*>(scratch(ctx->idx_d, std::max(p, 1)));
    CK(cudaMemcpyAsync(Aw, X->d(), sizeof(double) * (size_t)N * p, cudaMemcpyDeviceToDevice,
                       ctx->stream));
    if (launch_qr(Aw, N, n, p, tau, jpvt, vn, vn + p, ctx->stream) != 0)
        throw Fail{FL_CUDA, "colpiv_qr: cooperative launch failed"};
    g_launch_count += 1;
    std::vector<double> diag(kmax);
    CK(cudaMemcpy2DAsync(diag.data(), sizeof(double), Aw, sizeof(double) * (N + 1), sizeof(double),
                         kmax, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    double maxpivot = 0.0;
    for (double d : diag) maxpivot = std::max(maxpivot, std::abs(d));
    int r = 0;
    for (double d : diag)
        if (std::abs(d) > maxpivot * thr) ++r;
    if (U && r > 0) {
        block_reserve(U, r);
        block_set_cols(U, r);
        if (launch_orgqr(Aw, N, tau, n, r, U->d(), U->ld(), ctx->stream) != 0)
            throw Fail{FL_CUDA, "colpiv_qr: cooperative launch failed"};
        g_launch_count += 1;
        sync(ctx);
    }
    return r;
}

void orthonormalize_dev(fl_ctx* ctx, const fl_block* X, double drop_tol, fl_block* U, int* rank_out) {
    Prof pr(ctx, P_ORTH, (double)X->cols, 0);
    const int p = X->cols, N = X->N, n = X->n;
    if (p < 1 || n < 1) throw Fail{FL_INVALID_ARGUMENT, "orthonormalize: empty block"};
    const int P = round_up(p, FL_TILE);
    ensure_rr_scratch(ctx);
    double* G = scratch(ctx->s1, (size_t)P * P);
    double* Gs = scratch(ctx->s2, (size_t)P * P);
    double* work = scratch(ctx->s3, (size_t)P * P);
    double* V = scratch(ctx->s4, (size_t)P * P);
    double* Vt = scratch(ctx->s5, (size_t)P * P);
    double* vals = scratch(ctx->vals_d, P);
    // G = X^T X (ritz.cpp:32), symmetrised (:33)
    DGemm g{P, P, N, X->d(), X->ld(), 0, X->d(), X->ld(), 0, G, P, 0, 1.0, 0.0};
    launch_dgemm(g, true, false, 1, ctx->stream);
    launch_symmetrize(G, P, p, Gs, P, ctx->stream);
    g_launch_count += 2;
    device_sym_eig(ctx, Gs, P, p, P, vals, V, work, Vt);  // ascending (:34-35)
    std::vector<double> ev(p);
    CK(cudaMemcpyAsync(ev.data(), vals, sizeof(double) * p, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    // host decision logic, verbatim (ritz.cpp:36-51)
    const double sigma_max = std::sqrt(std::max(0.0, ev[p - 1]));
    if (!(sigma_max > 0.0)) throw Fail{FL_RUNTIME_ERROR, "orthonormalize: block is numerically zero"};
    const double ev_floor =
        std::max(drop_tol * drop_tol, std::numeric_limits<double>::epsilon() * p) * ev[p - 1];
    std::vector<int> keep;
    for (int i = p - 1; i >= 0; --i)
        if (ev[i] > ev_floor) keep.push_back(i);
    const int rank = (int)keep.size();
    if (g_decision_log.load()) {
        // the Gram-floor rank decision (ritz.cpp:44-49): the kept and dropped
        // eigenvalues next to the floor, and the eigensolver's absolute error
        // scale eps * ev_max, all relative to the floor
        const double eps = std::numeric_limits<double>::epsilon();
        const double kept_min = rank > 0 ? ev[p - rank] : 0.0;
        const double drop_max = rank < p ? ev[p - rank - 1] : 0.0;
        int near = 0;  // eigenvalues within 8 eps ev_max of the floor: undecidable
        for (int i = 0; i < p; ++i)
            if (std::abs(ev[i] - ev_floor) <= 8.0 * eps * ev[p - 1]) ++near;
        std::fprintf(stderr,
                     "decision gram_floor p=%d rank=%d kept_min/floor=%.6f dropped_max/floor=%.6f "
                     "eps*ev_max/floor=%.3e within_8eps=%d\n",
                     p, rank, kept_min / ev_floor, drop_max / ev_floor, eps * ev[p - 1] / ev_floor, near);
    }
    if (rank == 0) throw Fail{FL_RUNTIME_ERROR, "orthonormalize: block is numerically zero"};
    const int RP = round_up(rank, FL_TILE);
    // Vk = V[:, keep] (zero padded), U = X Vk, U[:, j] /= sigma_j (:53-57)
    std::vector<double> sig(rank);
    for (int j = 0; j < rank; ++j) sig[j] = std::sqrt(ev[keep[j]]);
    int* idx = reinterpret_cast<int*>(scratch(ctx->idx_d, rank));
    double* sg = scratch(ctx->norms_d, rank);
    CK(cudaMemcpyAsync(idx, keep.data(), sizeof(int) * rank, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(sg, sig.data(), sizeof(double) * rank, cudaMemcpyHostToDevice, ctx->stream));
    double* Vk = Vt;  // reuse
    launch_gather_cols(V, P, P, idx, rank, RP, Vk, P, ctx->stream);
    block_reserve(U, rank);
    block_set_cols(U, rank);
    DGemm h{N, RP, P, X->d(), X->ld(), 0, Vk, P, 0, U->d(), U->ld(), 0, 1.0, 0.0};
    launch_dgemm(h, false, false, 1, ctx->stream);
    launch_col_div(U->d(), U->ld(), n, rank, sg, ctx->stream);
    g_launch_count += 3;
    U->dirty = std::max(U->dirty, RP);
    block_set_cols(U, rank);
    sync(ctx);  // host vectors (keep, sig) go out of scope
    *rank_out = rank;
}

__global__ void transpose_kernel(const double* __restrict__ M, long ldm, int P, double* T, long ldt) {
    const long total = (long)P * P;
    for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long)gridDim.x * blockDim.x) {
        const int j = (int)(e / P), i = (int)(e - (long)j * P);
        T[(long)j * ldt + i] = M[(long)i * ldm + j];
    }
}

struct RRResult {
    std::vector<double> vals, norms;
    std::vector<unsigned char> inside;
};

void rayleigh_ritz_dev(fl_ctx* ctx, const fl_matrix* A, const fl_block* X, double lo, double hi,
                       fl_block* Vout, RRResult& out) {
    Prof pr(ctx, P_RR, (double)X->cols, 0);
    const int p = X->cols, N = X->N, n = X->n;
    if (n != A->n) throw Fail{FL_INVALID_ARGUMENT, "rayleigh_ritz: block/matrix dimension mismatch"};
    if (p < 1) throw Fail{FL_INVALID_ARGUMENT, "rayleigh_ritz: empty block"};
    const int P = round_up(p, FL_TILE);
    ensure_rr_scratch(ctx);
    double* AX = scratch(ctx->rr_nxp, (size_t)N * P);
    double* Ap = scratch(ctx->s1, (size_t)P * P);
    double* Bp = scratch(ctx->s2, (size_t)P * P);
    double* Aps = scratch(ctx->s3, (size_t)P * P);
    double* L = scratch(ctx->s4, (size_t)P * P);
    double* C = scratch(ctx->s5, (size_t)P * P);
    double* V = scratch(ctx->s6, (size_t)P * P);
    double* Vt = scratch(ctx->s7, (size_t)P * P);
    double* vals = scratch(ctx->vals_d, P);
    double* nrm = scratch(ctx->norms_d, P);
    cudaStream_t s = ctx->stream;
    // AX = A X ; A' = X^T AX ; B' = X^T X (ritz.cpp:90-92)
    launch_dgemm(DGemm{N, P, N, A->d(), N, 0, X->d(), X->ld(), 0, AX, N, 0, 1.0, 0.0}, false, false, 1, s);
    launch_dgemm(DGemm{P, P, N, X->d(), X->ld(), 0, AX, N, 0, Ap, P, 0, 1.0, 0.0}, true, false, 1, s);
    launch_dgemm(DGemm{P, P, N, X->d(), X->ld(), 0, X->d(), X->ld(), 0, Bp, P, 0, 1.0, 0.0}, true, false, 1, s);
    // symmetrise (:93-94) into zero-padded buffers; B' padded with identity
    CK(cudaMemsetAsync(Aps, 0, sizeof(double) * (size_t)P * P, s));
    CK(cudaMemsetAsync(L, 0, sizeof(double) * (size_t)P * P, s));
    launch_symmetrize(Ap, P, p, Aps, P, s);
    launch_symmetrize(Bp, P, p, L, P, s);
    launch_set_diag(L, P, p, P, 1.0, s);
    // L = chol(B') with the first failing pivot (:96, :64-79)
    int init[4] = {-1, 0, 0, 0};
    CK(cudaMemcpyAsync(ctx->chol_info.p, init, 16, cudaMemcpyHostToDevice, s));
    launch_cholesky(L, P, p, P, ctx->chol_info.p, s);
    struct {
        int index;
        double pivot;
    } info;
    CK(cudaMemcpyAsync(&info, ctx->chol_info.p, sizeof(info), cudaMemcpyDeviceToHost, s));
    sync(ctx);
    g_launch_count += 8 + 3 * (P / 64);
    if (info.index >= 0) {
        char buf[160];
        std::snprintf(buf, sizeof(buf), "rayleigh_ritz: B' not numerically SPD, pivot %f at index %d",
                      info.pivot, info.index);
        Fail f{FL_CHOLESKY, buf};
        f.index = info.index;
        f.pivot = info.pivot;
        throw f;
    }
    launch_tril(L, P, P, s);
    // T = L^{-1} A' (:97) ; C = L^{-1} T^T (:98) ; symmetrise (:99)
    launch_trsm_lower(L, P, P, Aps, P, P, false, s);
    transpose_kernel<<<148, 256, 0, s>>>(Aps, P, P, C, P);
    launch_trsm_lower(L, P, P, C, P, P, false, s);
    CK(cudaMemsetAsync(Ap, 0, sizeof(double) * (size_t)P * P, s));
    launch_symmetrize(C, P, p, Ap, P, s);
    g_launch_count += 3 + 4 * (P / 64);
    // eig (:101), Q = L^{-T} V (:102-103)
    device_sym_eig(ctx, Ap, P, p, P, vals, V, C, Vt);
    launch_trsm_lower(L, P, P, V, P, P, true, s);
    // vectors = X Q (:107)
    block_reserve(Vout, p);
    block_set_cols(Vout, p);
    launch_dgemm(DGemm{N, P, P, X->d(), X->ld(), 0, V, P, 0, Vout->d(), Vout->ld(), 0, 1.0, 0.0},
                 false, false, 1, s);
    Vout->dirty = std::max(Vout->dirty, P);
    block_set_cols(Vout, p);
    // unit-normalise (:110-112)
    launch_col_norms(Vout->d(), Vout->ld(), n, p, nrm, s);
    launch_col_div(Vout->d(), Vout->ld(), n, p, nrm, s);
    // R = A V - V diag(lam) (:115), norms (:116)
    launch_dgemm(DGemm{N, P, N, A->d(), N, 0, Vout->d(), Vout->ld(), 0, AX, N, 0, 1.0, 0.0}, false,
                 false, 1, s);
    double* R = scratch(ctx->rr_nxp2, (size_t)N * P);
    launch_residual(AX, N, Vout->d(), Vout->ld(), n, p, vals, R, N, s);
    launch_col_norms(R, N, n, p, nrm, s);
    g_launch_count += 7 + 2 * (P / 64);
    out.vals.resize(p);
    out.norms.resize(p);
    out.inside.resize(p);
    CK(cudaMemcpyAsync(out.vals.data(), vals, sizeof(double) * p, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(out.norms.data(), nrm, sizeof(double) * p, cudaMemcpyDeviceToHost, s));
    sync(ctx);
    for (int k = 0; k < p; ++k) out.inside[k] = (out.vals[k] > lo && out.vals[k] < hi) ? 1 : 0;
    if (g_decision_log.load()) {
        // the inside test (ritz.cpp:108-112): the Ritz value nearest to an interval
        // edge, relative to the interval's half width, and that pair's residual
        double best = 1e300, res = 0.0;
        int m = 0;
        for (int k = 0; k < p; ++k) {
            m += out.inside[k];
            const double d = std::min(std::abs(out.vals[k] - lo), std::abs(out.vals[k] - hi));
            if (d < best) {
                best = d;
                res = out.norms[k];
            }
        }
        std::fprintf(stderr, "decision inside p=%d m=%d nearest_edge_distance/radius=%.3e its_residual=%.3e\n",
                     p, m, best / (0.5 * (hi - lo)), res);
    }
}

template <class F>
int guarded(fl_err* err, F&& body) {
    try {
        body();
        return FL_OK;
    } catch (const Fail& f) {
        return report(err, f);
    } catch (const LaunchError& e) {
        return report(err, Fail{FL_CUDA, e.what()});
    } catch (const std::bad_alloc&) {
        return report(err, Fail{FL_OOM, "host allocation failed"});
    } catch (const std::exception& e) {
        return report(err, Fail{FL_RUNTIME_ERROR, e.what()});
    }
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

int fl_version(void) { return 1; }

int fl_device_count(int* count) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    *count = (e == cudaSuccess) ? c : 0;
    return e == cudaSuccess ? FL_OK : FL_CUDA;
}

static int ctx_create_impl(int device, const void* id, int rank, int nranks, fl_ctx** out,
                           fl_err* err) {
    return guarded(err, [&] {
        int cnt = 0;
        if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt == 0)
            throw Fail{FL_CUDA, "no CUDA device: the feastlab B200 path has no CPU fallback"};
        if (device < 0 || device >= cnt) throw Fail{FL_INVALID_ARGUMENT, "bad device index"};
        std::unique_ptr<fl_ctx> c(new fl_ctx());
        c->device = device;
        CK(cudaSetDevice(device));
        CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        const int naux = 8;
        int prio_lo = 0, prio_hi = 0;
        CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        c->aux.resize(naux);
        c->paux.resize(naux);
        c->join.resize(naux);
        c->ev_panel.resize(naux);
        c->ev_next.resize(naux);
        for (int j = 0; j < naux; ++j) {
            CK(cudaStreamCreateWithFlags(&c->aux[j], cudaStreamNonBlocking));
            // panels are the critical path: highest priority
            const char* pe = std::getenv("FEASTLAB_PANEL_PRIO");
            CK(cudaStreamCreateWithPriority(&c->paux[j], cudaStreamNonBlocking,
                                            (pe && pe[0] == '0') ? prio_lo : prio_hi));
            CK(cudaEventCreateWithFlags(&c->join[j], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&c->ev_panel[j], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&c->ev_next[j], cudaEventDisableTiming));
        }
        CK(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming));
        CK(cudaMallocHost(&c->h_cnt, sizeof(unsigned long long)));
        c->rank = rank;
        c->nranks = nranks;
        if (const char* fe = std::getenv("FEASTLAB_FACTOR"))
            c->factorization = std::strcmp(fe, "ldlt") == 0 ? FL_FACTOR_LDLT : FL_FACTOR_LU;
        if (id != nullptr) {  // a clique (also of one rank: exercises the NCCL path)
            ncclUniqueId uid;
            std::memcpy(&uid, id, sizeof(uid));
            nccl_check(ncclCommInitRank(&c->comm, nranks, uid, rank), "ncclCommInitRank");
        }
        c->launches_at_create = g_launch_count.load();
        *out = c.release();
    });
}

int fl_ctx_create(int device, fl_ctx** out, fl_err* err) {
    return ctx_create_impl(device, nullptr, 0, 1, out, err);
}

int fl_ctx_create_nccl(int device, const void* nccl_id, int rank, int nranks, fl_ctx** out,
                       fl_err* err) {
    if (nranks < 1 || rank < 0 || rank >= nranks || nccl_id == nullptr)
        return report(err, Fail{FL_INVALID_ARGUMENT, "bad rank/nranks or missing NCCL id"});
    return ctx_create_impl(device, nccl_id, rank, nranks, out, err);
}

int fl_ctx_create_virtual(int device, int rank, int nranks, fl_ctx** out, fl_err* err) {
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return report(err, Fail{FL_INVALID_ARGUMENT, "bad rank/nranks"});
    return ctx_create_impl(device, nullptr, rank, nranks, out, err);
}

int fl_nccl_unique_id(void* out128, fl_err* err) {
    return guarded(err, [&] {
        ncclUniqueId uid;
        nccl_check(ncclGetUniqueId(&uid), "ncclGetUniqueId");
        std::memcpy(out128, &uid, sizeof(uid));
    });
}

static void ctx_teardown(fl_ctx* ctx) {
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->comm) ncclCommDestroy(ctx->comm);
    for (cudaStream_t a : ctx->aux) {
        cudaStreamSynchronize(a);
        cudaStreamDestroy(a);
    }
    for (cudaEvent_t e : ctx->join) cudaEventDestroy(e);
    for (cudaStream_t a : ctx->paux) {
        cudaStreamSynchronize(a);
        cudaStreamDestroy(a);
    }
    for (cudaEvent_t e : ctx->ev_panel) cudaEventDestroy(e);
    for (cudaEvent_t e : ctx->ev_next) cudaEventDestroy(e);
    if (ctx->fork) cudaEventDestroy(ctx->fork);
    if (ctx->done) cudaEventDestroy(ctx->done);
    if (ctx->h_cnt) cudaFreeHost(ctx->h_cnt);
    cudaStreamDestroy(ctx->stream);
    delete ctx;
}

static void ctx_retain(fl_ctx* ctx) { ctx->refs.fetch_add(1); }

static void ctx_release(fl_ctx* ctx) {
    if (ctx->refs.fetch_sub(1) == 1) ctx_teardown(ctx);
}

int fl_ctx_destroy(fl_ctx* ctx) {
    if (ctx) ctx_release(ctx);
    return FL_OK;
}

int fl_ctx_sync(fl_ctx* ctx, fl_err* err) {
    return guarded(err, [&] {
        CtxLock lk(ctx);
        sync(ctx);
    });
}

void* fl_ctx_stream(fl_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int fl_ctx_rank(const fl_ctx* ctx, int* rank, int* nranks) {
    *rank = ctx->rank;
    *nranks = ctx->nranks;
    return FL_OK;
}

long long fl_ctx_launches(const fl_ctx* ctx) { return g_launch_count.load() - ctx->launches_at_create; }

// timeline of the profiled launches: out[5*i] = class, [5*i+1] = start ms,
// [5*i+2] = end ms (relative to the first recorded event), [5*i+3] = work,
// [5*i+4] = shape tag (GEMM classes, shape_tag(); else 0); returns the count
int fl_ctx_profile_dump(fl_ctx* ctx, double* out, int max_records) {
    CtxLock lk(ctx);
    cudaStreamSynchronize(ctx->stream);
    cudaDeviceSynchronize();
    const auto& recs = ctx->prof.recs;
    if (recs.empty()) return 0;
    const cudaEvent_t base = recs[0].a;
    int n = 0;
    for (const auto& r : recs) {
        if (n >= max_records) break;
        float a = 0.f, b = 0.f;
        cudaEventElapsedTime(&a, base, r.a);
        cudaEventElapsedTime(&b, base, r.b);
        out[5 * n] = r.cls;
        out[5 * n + 1] = a;
        out[5 * n + 2] = b;
        out[5 * n + 3] = r.work;
        out[5 * n + 4] = r.tag;
        ++n;
    }
    return n;
}

// microbenchmark of the planar-complex DMMA GEMM (C -= A B, batch x M x N x K,
// operands resident in HBM): average milliseconds per launch
int fl_debug_zgemm(fl_ctx* ctx, int M, int Nc, int K, int batch, int iters, double* ms_out,
                   fl_err* err) {
    return guarded(err, [&] {
        CtxLock lk(ctx);
        if (M % 64 || Nc % 64 || K % 16 || batch < 1 || iters < 1)
            throw Fail{FL_INVALID_ARGUMENT, "fl_debug_zgemm: bad shape"};
        const size_t a = (size_t)M * K, b = (size_t)K * Nc, c = (size_t)M * Nc;
        DBuf buf;
        buf.ensure(sizeof(double) * 2 * (a + b + c) * batch);
        CK(cudaMemsetAsync(buf.p, 0, sizeof(double) * 2 * (a + b + c) * batch, ctx->stream));
        double* base = buf.d();
        const long sa = 2 * a, sb = 2 * b, sc = 2 * c;
        ZGemm g{M, Nc, K, base, base + a, M, sa, base + sa * batch, base + sa * batch + b, K, sb,
                base + (sa + sb) * batch, base + (sa + sb) * batch + c, M, sc};
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        launch_zgemm_sub(g, batch, ctx->stream);
        cudaEventRecord(e0, ctx->stream);
        for (int i = 0; i < iters; ++i) launch_zgemm_sub(g, batch, ctx->stream);
        cudaEventRecord(e1, ctx->stream);
        CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *ms_out = ms / iters;
    });
}

// The same product in the LU's own layout: batch N x N planar factors,
// C = F[N-M:, N-M : N-M+Nc] -= F[N-M:, 0:K] F[0:K, N-M : N-M+Nc] (ld N, so the
// operand tiles are strided exactly as in a trailing update). The planes hold
// pseudo-random values; *checksum = sum of C after one product from the
// initial fill (to compare kernel variants bit for bit).
namespace {
__global__ void debug_fill_kernel(double* p, size_t n, unsigned seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        unsigned long long x = (i + 1) * 0x9E3779B97F4A7C15ull + seed * 0xD1B54A32D192ED03ull;
        x ^= x >> 29;
        x *= 0xBF58476D1CE4E5B9ull;
        x ^= x >> 32;
        p[i] = ((double)(x >> 11) * (1.0 / 9007199254740992.0) - 0.5) * 0.0625;
    }
}
__global__ void debug_sum_kernel(const double* re, const double* im, long ld, int M, int Nc,
                                 long stride, int batch, double* out) {
    double s = 0.0;
    const long total = (long)M * Nc * batch;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total;
         i += (long)gridDim.x * blockDim.x) {
        const long b = i / ((long)M * Nc), r = i % ((long)M * Nc);
        const long off = b * stride + (r / M) * ld + (r % M);
        s += re[off] * 1.0 + im[off] * 0.5;
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, s);
}
}  // namespace

__global__ void debug_maxdiff_kernel(const double* a, const double* b, size_t n, double* out) {
    double d = 0.0, m = 0.0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x) {
        d = fmax(d, fabs(a[i] - b[i]));
        m = fmax(m, fabs(a[i]));
    }
    for (int off = 16; off > 0; off >>= 1) {
        d = fmax(d, __shfl_xor_sync(0xffffffffu, d, off));
        m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    }
    if ((threadIdx.x & 31) == 0) {  // non-negative doubles order as their bit patterns
        atomicMax(reinterpret_cast<unsigned long long*>(out), (unsigned long long)__double_as_longlong(d));
        atomicMax(reinterpret_cast<unsigned long long*>(out + 1), (unsigned long long)__double_as_longlong(m));
    }
}

int fl_debug_zgemm_lu(fl_ctx* ctx, int N, int M, int Nc, int K, int batch, int iters, int variant,
                      double* ms_out, double* checksum, double* maxdiff, fl_err* err) {
    return guarded(err, [&] {
        CtxLock lk(ctx);
        if (N % 64 || M % 64 || Nc % 64 || K % 16 || batch < 1 || iters < 1 || M + K > N ||
            Nc > M)
            throw Fail{FL_INVALID_ARGUMENT, "fl_debug_zgemm_lu: bad shape"};
        const size_t plane = (size_t)N * N;
        DBuf buf, ref, sum, sa, sb;
        buf.ensure(sizeof(double) * 2 * plane * batch);
        sum.ensure(sizeof(double) * 4);
        double* re = buf.d();
        double* im = re + plane * batch;
        auto fill = [&] {
            debug_fill_kernel<<<148 * 8, 256, 0, ctx->stream>>>(re, 2 * plane * batch, 17u);
        };
        const int c0 = N - M;
        auto E = [&](int r, int c) { return (long)c * N + r; };
        ZGemm g{M, Nc, K, re + E(c0, 0), im + E(c0, 0), N, (long)plane,
                re + E(0, c0), im + E(0, c0), N, (long)plane,
                re + E(c0, c0), im + E(c0, c0), N, (long)plane};
        ZGemmMaps maps;
        ZGemmTma t{M, Nc, K, c0, 0, 0, c0, 0, 0, 0, c0, 0, 0, c0, 0, g.Cr, g.Ci, N, (long)plane};
        if (variant >= 1) {
            sa.ensure(sizeof(double) * (size_t)N * K * batch);
            sb.ensure(sizeof(double) * (size_t)K * N * batch);
            make_tma_map_mk(&maps.Ar, re, N, N, N, (long)plane, batch);
            make_tma_map_mk(&maps.Ai, im, N, N, N, (long)plane, batch);
            make_tma_map_mk(&maps.As, sa.d(), N, K, N, (long)N * K, batch);
            make_tma_map_km(&maps.Br, re, N, N, N, (long)plane, batch);
            make_tma_map_km(&maps.Bi, im, N, N, N, (long)plane, batch);
            make_tma_map_km(&maps.Bs, sb.d(), K, N, K, (long)K * N, batch);
        }
        auto sums = [&] {
            launch_zsum(re + E(c0, 0), im + E(c0, 0), N, (long)plane, sa.d() + c0, N, (long)N * K, M,
                        K, batch, ctx->stream);
            launch_zsum(re + E(0, c0), im + E(0, c0), N, (long)plane, sb.d() + (long)c0 * K, K,
                        (long)K * N, K, Nc, batch, ctx->stream);
        };
        auto run = [&](int v) {
            if (v == 1) {
                launch_zgemm_sub_tma(maps, t, batch, ctx->stream);
            } else {
                launch_zgemm_sub(g, batch, ctx->stream);
            }
        };
        fill();
        if (variant >= 1) sums();
        run(variant);
        CK(cudaMemsetAsync(sum.p, 0, sizeof(double) * 4, ctx->stream));
        debug_sum_kernel<<<148 * 4, 256, 0, ctx->stream>>>(g.Cr, g.Ci, N, M, Nc, (long)plane,
                                                          batch, sum.d());
        double host[4] = {0, 0, 0, 0};
        if (variant != 0 && maxdiff) {  // against the cp.async kernel on the same fill
            ref.ensure(sizeof(double) * 2 * plane * batch);
            CK(cudaMemcpyAsync(ref.p, buf.p, sizeof(double) * 2 * plane * batch,
                               cudaMemcpyDeviceToDevice, ctx->stream));
            fill();
            run(0);
            debug_maxdiff_kernel<<<148 * 4, 256, 0, ctx->stream>>>(re, ref.d(), 2 * plane * batch,
                                                              sum.d() + 1);
        }
        CK(cudaMemcpyAsync(host, sum.p, sizeof(double) * 4, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        if (checksum) *checksum = host[0];
        if (maxdiff) {
            maxdiff[0] = host[1];
            maxdiff[1] = host[2];
        }
        ref.release();
        fill();
        if (variant >= 1) sums();
        run(variant);  // warm
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, ctx->stream);
        for (int i = 0; i < iters; ++i) run(variant);
        cudaEventRecord(e1, ctx->stream);
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *ms_out = ms / iters;
    });
}

namespace {
__global__ void tile_sums_kernel(const double* re, const double* im, long ld, long stride, int NB,
                                 double* out) {
    const int tr = blockIdx.x, tc = blockIdx.y, b = blockIdx.z;
    const double* r = re + b * stride + (long)tc * 64 * ld + tr * 64;
    const double* i = im + b * stride + (long)tc * 64 * ld + tr * 64;
    double s = 0.0;
    for (int e = threadIdx.x; e < 4096; e += blockDim.x) {
        const long o = (long)(e >> 6) * ld + (e & 63);
        s += r[o] * (1.0 + 1e-3 * (e & 63)) + i[o] * (0.5 + 1e-3 * (e >> 6));
    }
    __shared__ double sh[8];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < blockDim.x / 32; ++w) t += sh[w];
        out[((long)b * NB + tc) * NB + tr] = t;
    }
}
}  // namespace

// weighted sums of the 64 x 64 tiles of the factor in slots [0, count) (out:
// count x NB x NB, tile column-major) -- compares factorizations across runs
int fl_debug_factor_tilesums(fl_filter* f, int count, double* out) {
    fl_ctx* ctx = f->ctx;
    CtxLock lk(ctx);
    const int N = f->A->N, NB = N / FL_TILE;
    if (count > f->fac_slots) return FL_INVALID_ARGUMENT;
    DBuf d;
    d.ensure(sizeof(double) * (size_t)count * NB * NB);
    cudaStreamSynchronize(ctx->stream);
    tile_sums_kernel<<<dim3(NB, NB, count), 256, 0, ctx->stream>>>(f->fac_re.d(), f->fac_im.d(), N,
                                                                   (long)N * N, NB, d.d());
    cudaMemcpyAsync(out, d.p, sizeof(double) * (size_t)count * NB * NB, cudaMemcpyDeviceToHost,
                    ctx->stream);
    return cudaStreamSynchronize(ctx->stream) == cudaSuccess ? FL_OK : FL_CUDA;
}

// ---------------------------------------------------------------- fixtures
// seeded_orthogonal of proj/src/matmodel.cpp:93-105 on the device: Householder
// QR of the n x n block G (column-major, ld n), Q = H_1 ... H_n I, columns
// sign-normalised. G and Q: host or device (loc_*), Q ld n.
int fl_fixture_orthogonal(fl_ctx* ctx, const double* G, int n, int loc_g, double* Q, int loc_q,
                          fl_err* err) {
    return guarded(err, [&] {
        if (n < 1) throw Fail{FL_INVALID_ARGUMENT, "fl_fixture_orthogonal: need n >= 1"};
        CtxLock lk(ctx);
        const int N = round_up(n, FL_TILE);
        DBuf a, q, v, w, w2, g, t, tau;
        a.ensure(sizeof(double) * (size_t)N * N);
        q.ensure(sizeof(double) * (size_t)N * N);
        v.ensure(sizeof(double) * (size_t)N * FL_TILE);
        w.ensure(sizeof(double) * (size_t)N * FL_TILE);
        w2.ensure(sizeof(double) * (size_t)N * FL_TILE);
        g.ensure(sizeof(double) * FL_TILE * FL_TILE);
        t.ensure(sizeof(double) * (size_t)N * FL_TILE);
        tau.ensure(sizeof(double) * N);
        CK(cudaMemsetAsync(a.p, 0, sizeof(double) * (size_t)N * N, ctx->stream));
        copy_in(ctx, a.d(), N, n, G, n, n, loc_g);
        launch_set_diag(a.d(), N, n, N, 1.0, ctx->stream);  // identity padding block
        if (fixture_householder_q(a.d(), N, q.d(), v.d(), w.d(), w2.d(), g.d(), t.d(), tau.d(),
                                  ctx->stream) != 0)
            throw Fail{FL_CUDA, "fl_fixture_orthogonal: launch failed"};
        fixture_sign_normalize(q.d(), N, n, ctx->stream);
        g_launch_count += 4 + 10LL * (N / FL_TILE);
        copy_out(ctx, Q, n, n, q.d(), N, n, loc_q);
        sync(ctx);
    });
}

// assemble_matrix of proj/src/matmodel.cpp:109-118: A = 0.5 (M + M^T),
// M = Q diag(vals) Q^T. Q (ld n) and A (ld n, may be Q): host or device; vals: host.
int fl_fixture_assemble(fl_ctx* ctx, const double* Q, int loc_q, const double* vals, int n,
                        double* A, int loc_a, fl_err* err) {
    return guarded(err, [&] {
        if (n < 1) throw Fail{FL_INVALID_ARGUMENT, "fl_fixture_assemble: need n >= 1"};
        CtxLock lk(ctx);
        const int N = round_up(n, FL_TILE);
        DBuf q, b, m, a, vd;
        q.ensure(sizeof(double) * (size_t)N * N);
        b.ensure(sizeof(double) * (size_t)N * N);
        m.ensure(sizeof(double) * (size_t)N * N);
        a.ensure(sizeof(double) * (size_t)N * N);
        vd.ensure(sizeof(double) * N);
        CK(cudaMemsetAsync(q.p, 0, sizeof(double) * (size_t)N * N, ctx->stream));
        copy_in(ctx, q.d(), N, n, Q, n, n, loc_q);
        CK(cudaMemcpyAsync(vd.p, vals, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
        fixture_assemble(q.d(), vd.d(), N, n, b.d(), m.d(), a.d(), ctx->stream);
        g_launch_count += 3;
        copy_out(ctx, A, n, n, a.d(), N, n, loc_a);
        sync(ctx);
    });
}

int fl_debug_decision_log(int on) {
    if (on >= 0) g_decision_log.store(on ? 1 : 0);
    return g_decision_log.load();
}

int fl_ctx_set_reduction(fl_ctx* ctx, int mode) {
    if (!ctx || (mode != FL_REDUCE_SUM && mode != FL_REDUCE_ORDERED)) return FL_INVALID_ARGUMENT;
    CtxLock lk(ctx);
    ctx->reduction = mode;
    return FL_OK;
}

int fl_ctx_set_factorization(fl_ctx* ctx, int mode) {
    if (!ctx || (mode != FL_FACTOR_LU && mode != FL_FACTOR_LDLT)) return FL_INVALID_ARGUMENT;
    CtxLock lk(ctx);
    ctx->factorization = mode;
    return FL_OK;
}

int fl_ctx_factorization(const fl_ctx* ctx) { return ctx ? ctx->factorization : -1; }

int fl_zgemm_mode(int mode) {
    if (mode >= 0) set_zgemm_mode(mode);
    return zgemm_mode();
}

int fl_debug_panel_profile(double* out8, int reset) {
    panel_profile(out8, reset != 0);
    return FL_OK;
}

int fl_debug_panel_trace(long long* out, int max) { return fl::res_panel_trace(out, max); }

int fl_ctx_set_streams(fl_ctx* ctx, int n) {
    CtxLock lk(ctx);
    ctx->nstreams = std::max(1, std::min(n, (int)ctx->aux.size()));
    return FL_OK;
}

int fl_ctx_set_profiling(fl_ctx* ctx, int on) {
    CtxLock lk(ctx);
    ctx->prof.on = on != 0;
    ctx->prof.reset();
    return FL_OK;
}

int fl_ctx_profile(fl_ctx* ctx, const char* cls, double* ms, double* work, long long* launches,
                   fl_err* err) {
    return guarded(err, [&] {
        CtxLock lk(ctx);
        int k = -1;
        for (int i = 0; i < P_NCLASS; ++i)
            if (std::strcmp(cls, kProfNames[i]) == 0) k = i;
        if (k < 0) throw Fail{FL_INVALID_ARGUMENT, std::string("unknown kernel class ") + cls};
        sync(ctx);
        double t = 0.0, w = 0.0;
        long long c = 0;
        for (const auto& r : ctx->prof.recs) {
            if (r.cls != k) continue;
            float e = 0.f;
            CK(cudaEventElapsedTime(&e, r.a, r.b));
            t += e;
            w += r.work;
            ++c;
        }
        *ms = t;
        *work = w;
        *launches = c;
    });
}

int fl_matrix_create(fl_ctx* ctx, const double* A, int n, int lda, int loc, fl_matrix** out,
                     fl_err* err) {
    return guarded(err, [&] {
        if (n < 1 || lda < n) throw Fail{FL_INVALID_ARGUMENT, "fl_matrix_create: bad shape"};
        CtxLock lk(ctx);
        std::unique_ptr<fl_matrix> m(new fl_matrix());
        m->ctx = ctx;
        m->n = n;
        m->N = round_up(n, FL_TILE);
        m->buf.ensure(sizeof(double) * (size_t)m->N * m->N);
        CK(cudaMemsetAsync(m->buf.p, 0, sizeof(double) * (size_t)m->N * m->N, ctx->stream));
        // a device-resident A may still be in flight on the producer's stream
        // (e.g. torch's): the one-time copy waits for the whole device
        if (loc == FL_DEVICE) CK(cudaDeviceSynchronize());
        copy_in(ctx, m->d(), m->N, n, A, lda, n, loc);
        sync(ctx);
        ctx_retain(ctx);
        *out = m.release();
    });
}

int fl_matrix_destroy(fl_matrix* m) {
    if (m) {
        fl_ctx* ctx = m->ctx;
        {
            CtxLock lk(ctx);
            delete m;
        }
        ctx_release(ctx);
    }
    return FL_OK;
}

int fl_matrix_dim(const fl_matrix* m) { return m->n; }

int fl_block_create(fl_ctx* ctx, int n, int cap_cols, fl_block** out, fl_err* err) {
    return guarded(err, [&] {
        if (n < 1 || cap_cols < 0) throw Fail{FL_INVALID_ARGUMENT, "fl_block_create: bad shape"};
        CtxLock lk(ctx);
        std::unique_ptr<fl_block> b(new fl_block());
        b->ctx = ctx;
        b->n = n;
        b->N = round_up(n, FL_TILE);
        block_reserve(b.get(), std::max(cap_cols, 1));
        ctx_retain(ctx);
        *out = b.release();
    });
}

int fl_block_destroy(fl_block* b) {
    if (b) {
        fl_ctx* ctx = b->ctx;
        {
            CtxLock lk(ctx);
            delete b;
        }
        ctx_release(ctx);
    }
    return FL_OK;
}

int fl_block_cols(const fl_block* b) { return b->cols; }
int fl_block_rows(const fl_block* b) { return b->n; }

int fl_block_set(fl_block* b, const double* X, int ldx, int p, int loc, fl_err* err) {
    return guarded(err, [&] {
        if (p < 0 || ldx < b->n) throw Fail{FL_INVALID_ARGUMENT, "fl_block_set: bad shape"};
        CtxLock lk(b->ctx);
        block_reserve(b, p);
        block_set_cols(b, p);
        copy_in(b->ctx, b->d(), b->ld(), b->n, X, ldx, p, loc);
        if (loc == FL_HOST) sync(b->ctx);
    });
}

int fl_block_get(const fl_block* b, double* X, int ldx, int loc, fl_err* err) {
    return guarded(err, [&] {
        if (ldx < b->n) throw Fail{FL_INVALID_ARGUMENT, "fl_block_get: bad ld"};
        CtxLock lk(b->ctx);
        copy_out(b->ctx, X, ldx, b->n, b->d(), b->ld(), b->cols, loc);
        if (loc == FL_HOST) sync(b->ctx);
    });
}

int fl_block_gather(fl_block* dst, const fl_block* src, const int* idx, int k, fl_err* err) {
    return guarded(err, [&] {
        if (dst == src) throw Fail{FL_INVALID_ARGUMENT, "fl_block_gather: dst aliases src"};
        if (dst->n != src->n) throw Fail{FL_INVALID_ARGUMENT, "fl_block_gather: row mismatch"};
        for (int j = 0; j < k; ++j)
            if (idx[j] < 0 || idx[j] >= src->cols)
                throw Fail{FL_INVALID_ARGUMENT, "fl_block_gather: index out of range"};
        fl_ctx* ctx = dst->ctx;
        CtxLock lk(ctx);
        block_reserve(dst, k);
        int* d_idx = reinterpret_cast<int*>(scratch(ctx->idx_d, std::max(k, 1)));
        if (k > 0)
            CK(cudaMemcpyAsync(d_idx, idx, sizeof(int) * k, cudaMemcpyHostToDevice, ctx->stream));
        const int kp = round_up(std::max(k, 1), FL_TILE);
        launch_gather_cols(src->d(), src->ld(), src->N, d_idx, k, std::min(kp, dst->CAP), dst->d(),
                           dst->ld(), ctx->stream);
        g_launch_count += 1;
        dst->dirty = std::max(dst->dirty, std::min(kp, dst->CAP));
        block_set_cols(dst, k);
        sync(ctx);
    });
}

int fl_block_append(fl_block* dst, const fl_block* src, fl_err* err) {
    return guarded(err, [&] {
        if (dst->n != src->n) throw Fail{FL_INVALID_ARGUMENT, "fl_block_append: row mismatch"};
        CtxLock lk(dst->ctx);
        const int c0 = dst->cols, k = src->cols;
        block_reserve(dst, c0 + k);
        if (k > 0)
            CK(cudaMemcpyAsync(dst->d() + (long)c0 * dst->ld(), src->d(),
                               sizeof(double) * (size_t)dst->ld() * k, cudaMemcpyDeviceToDevice,
                               dst->ctx->stream));
        dst->cols = c0 + k;
        dst->dirty = std::max(dst->dirty, dst->cols);
    });
}

int fl_block_copy(fl_block* dst, const fl_block* src, fl_err* err) {
    return guarded(err, [&] {
        if (dst->n != src->n) throw Fail{FL_INVALID_ARGUMENT, "fl_block_copy: row mismatch"};
        if (dst == src) return;
        CtxLock lk(dst->ctx);
        block_reserve(dst, src->cols);
        block_set_cols(dst, src->cols);
        if (src->cols > 0)
            CK(cudaMemcpyAsync(dst->d(), src->d(), sizeof(double) * (size_t)dst->ld() * src->cols,
                               cudaMemcpyDeviceToDevice, dst->ctx->stream));
    });
}

int fl_filter_create(fl_ctx* ctx, const fl_matrix* A, int n_c, const double* zr, const double* zi,
                     const double* wr, const double* wi, int cache, fl_filter** out, fl_err* err) {
    return guarded(err, [&] {
        if (n_c < 1) throw Fail{FL_INVALID_ARGUMENT, "fl_filter_create: need n_c >= 1"};
        std::unique_ptr<fl_filter> f(new fl_filter());
        f->ctx = ctx;
        f->A = A;
        f->nc = n_c;
        f->zr.assign(zr, zr + n_c);
        f->zi.assign(zi, zi + n_c);
        f->wr.assign(wr, wr + n_c);
        f->wi.assign(wi, wi + n_c);
        f->cache = cache != 0;
        // contiguous node shard of this rank
        fl_node_shard(n_c, ctx->rank, ctx->nranks, &f->kb, &f->ke);
        f->factored.assign(f->ke - f->kb, 0);
        ctx_retain(ctx);
        *out = f.release();
    });
}

int fl_filter_destroy(fl_filter* f) {
    if (f) {
        fl_ctx* ctx = f->ctx;
        {
            CtxLock lk(ctx);
            cudaStreamSynchronize(ctx->stream);  // in-flight verdict copy into f->h_bad
            auto& pend = ctx->pending;
            pend.erase(std::remove(pend.begin(), pend.end(), f), pend.end());
            delete f;
        }
        ctx_release(ctx);
    }
    return FL_OK;
}

int fl_filter_apply(fl_filter* f, const fl_block* X, fl_block* Y, long long* rhs, long long* facts,
                    fl_err* err) {
    return guarded(err, [&] {
        if (X->n != f->A->n)
            throw Fail{FL_INVALID_ARGUMENT, "apply_filter: block dimension " + std::to_string(X->n) +
                                                " != matrix dimension " + std::to_string(f->A->n)};
        if (X->cols < 1) throw Fail{FL_INVALID_ARGUMENT, "apply_filter: block must have p >= 1"};
        if (X == Y) throw Fail{FL_INVALID_ARGUMENT, "apply_filter: X and Y must differ"};
        CtxLock lk(f->ctx);
        block_reserve(Y, X->cols);
        block_set_cols(Y, X->cols);
        filter_apply_dev(f, X->d(), X->ld(), X->cols, Y->d(), Y->ld(), rhs, facts);
        Y->dirty = std::max(Y->dirty, round_up(X->cols, FL_TILE));
        block_set_cols(Y, X->cols);
    });
}

int fl_filter_apply_raw(fl_filter* f, const double* X, int ldx, int p, double* Y, int ldy, int loc,
                        long long* rhs, long long* facts, fl_err* err) {
    return guarded(err, [&] {
        const int n = f->A->n, N = f->A->N;
        if (p < 1) throw Fail{FL_INVALID_ARGUMENT, "apply_filter: block must have p >= 1"};
        if (ldx < n || ldy < n) throw Fail{FL_INVALID_ARGUMENT, "apply_filter: bad leading dimension"};
        fl_ctx* ctx = f->ctx;
        CtxLock lk(ctx);
        const int P = round_up(p, FL_TILE);
        // padded staging copies (zero rows >= n, zero cols >= p)
        double* Xs = scratch(f->y_tmp, (size_t)2 * N * P);
        double* Ys = Xs + (size_t)N * P;
        CK(cudaMemsetAsync(Xs, 0, sizeof(double) * (size_t)N * P, ctx->stream));
        copy_in(ctx, Xs, N, n, X, ldx, p, loc);
        if (loc == FL_DEVICE) {  // stays asynchronous: a singular node is raised by the next sync
            filter_apply_dev(f, Xs, N, p, Ys, N, rhs, facts);
            copy_out(ctx, Y, ldy, n, Ys, N, p, loc);
            return;
        }
        long long r = 0, fa = 0;
        filter_apply_dev(f, Xs, N, p, Ys, N, &r, &fa);
        copy_out(ctx, Y, ldy, n, Ys, N, p, loc);
        try {
            sync(ctx);
        } catch (const Fail& e) {
            // nodes factored before the singular one count (filterop.cpp:74-76)
            if (e.code == FL_SINGULAR_NODE && !f->cache && facts) *facts += e.index;
            throw;
        }
        if (rhs) *rhs += r;
        if (facts) *facts += fa;
    });
}

int fl_orthonormalize(fl_ctx* ctx, const fl_block* X, double drop_tol, int method, fl_block* U,
                      int* rank, fl_err* err) {
    return guarded(err, [&] {
        if (X->cols < 1 || X->n < 1) throw Fail{FL_INVALID_ARGUMENT, "orthonormalize: empty block"};
        if (X == U) throw Fail{FL_INVALID_ARGUMENT, "orthonormalize: X and U must differ"};
        CtxLock lk(ctx);
        if (method == 1) {
            const int r = colpiv_qr(ctx, X, drop_tol, U);
            if (r == 0) throw Fail{FL_RUNTIME_ERROR, "orthonormalize: block is numerically zero"};
            *rank = r;
        } else {
            orthonormalize_dev(ctx, X, drop_tol, U, rank);
        }
    });
}

int fl_rayleigh_ritz(fl_ctx* ctx, const fl_matrix* A, const fl_block* X, double lo, double hi,
                     double* vals, fl_block* V, double* norms, unsigned char* inside, fl_err* err) {
    return guarded(err, [&] {
        if (X == V) throw Fail{FL_INVALID_ARGUMENT, "rayleigh_ritz: X and V must differ"};
        CtxLock lk(ctx);
        RRResult r;
        rayleigh_ritz_dev(ctx, A, X, lo, hi, V, r);
        std::memcpy(vals, r.vals.data(), sizeof(double) * r.vals.size());
        std::memcpy(norms, r.norms.data(), sizeof(double) * r.norms.size());
        std::memcpy(inside, r.inside.data(), r.inside.size());
    });
}

int fl_residual_block(fl_ctx* ctx, const fl_matrix* A, const fl_block* V, const double* vals,
                      fl_block* R, fl_err* err) {
    return guarded(err, [&] {
        if (V->n != A->n) throw Fail{FL_INVALID_ARGUMENT, "compute_residual_block: dimension mismatch"};
        if (V == R) throw Fail{FL_INVALID_ARGUMENT, "compute_residual_block: V and R must differ"};
        CtxLock lk(ctx);
        const int p = V->cols, N = V->N, n = V->n;
        const int P = round_up(std::max(p, 1), FL_TILE);
        double* AV = scratch(ctx->rr_nxp, (size_t)N * P);
        double* lam = scratch(ctx->vals_d, P);
        if (p > 0)
            CK(cudaMemcpyAsync(lam, vals, sizeof(double) * p, cudaMemcpyHostToDevice, ctx->stream));
        launch_dgemm(DGemm{N, P, N, A->d(), N, 0, V->d(), V->ld(), 0, AV, N, 0, 1.0, 0.0}, false,
                     false, 1, ctx->stream);
        block_reserve(R, p);
        block_set_cols(R, p);
        launch_residual(AV, N, V->d(), V->ld(), n, p, lam, R->d(), R->ld(), ctx->stream);
        g_launch_count += 2;
        sync(ctx);
    });
}

int fl_block_rank(fl_ctx* ctx, const fl_block* X, double threshold, int* rank, fl_err* err) {
    return guarded(err, [&] {
        CtxLock lk(ctx);
        if (X->cols < 1) {
            *rank = 0;
            return;
        }
        *rank = colpiv_qr(ctx, X, threshold, nullptr);
    });
}

int fl_sym_eig(fl_ctx* ctx, const double* M, int p, int ldm, double* vals, double* V, int ldv,
               fl_err* err) {
    return guarded(err, [&] {
        if (p < 1 || ldm < p || ldv < p) throw Fail{FL_INVALID_ARGUMENT, "fl_sym_eig: bad shape"};
        CtxLock lk(ctx);
        const int P = round_up(p, FL_TILE);
        ensure_rr_scratch(ctx);
        double* Md = scratch(ctx->s1, (size_t)P * P);
        double* work = scratch(ctx->s3, (size_t)P * P);
        double* Vd = scratch(ctx->s4, (size_t)P * P);
        double* Vt = scratch(ctx->s5, (size_t)P * P);
        double* vd = scratch(ctx->vals_d, P);
        CK(cudaMemsetAsync(Md, 0, sizeof(double) * (size_t)P * P, ctx->stream));
        copy_in(ctx, Md, P, p, M, ldm, p, FL_HOST);
        device_sym_eig(ctx, Md, P, p, P, vd, Vd, work, Vt);
        CK(cudaMemcpyAsync(vals, vd, sizeof(double) * p, cudaMemcpyDeviceToHost, ctx->stream));
        copy_out(ctx, V, ldv, p, Vd, P, p, FL_HOST);
        sync(ctx);
    });
}

}  // extern "C"

struct fl_node {
    fl_ctx* ctx = nullptr;
    int node_index = -1;
    std::unique_ptr<fl_filter> f;
};

namespace {

// A one-node cached filter (weight 1) holding the factor of z I - A.
std::unique_ptr<fl_filter> node_filter(fl_ctx* ctx, const fl_matrix* A, double zr, double zi) {
    std::unique_ptr<fl_filter> f(new fl_filter());
    f->ctx = ctx;
    f->A = A;
    f->nc = 1;
    f->zr = {zr};
    f->zi = {zi};
    f->wr = {1.0};
    f->wi = {0.0};
    f->cache = true;
    f->kb = 0;
    f->ke = 1;
    f->factored.assign(1, 0);
    return f;
}

// W = S^{-1} (Br + i Bi) = S^{-1} Br + i S^{-1} Bi, both halves through the
// real-RHS path of the (cached) factor; B, W host interleaved complex n x p.
void node_solve_impl(fl_filter* f, const double* B, int p, double* W) {
    fl_ctx* ctx = f->ctx;
    const int n = f->A->n, N = f->A->N;
    const int P = round_up(2 * p, FL_TILE);
    DBuf X;
    X.ensure(sizeof(double) * (size_t)N * P);
    CK(cudaMemsetAsync(X.p, 0, sizeof(double) * (size_t)N * P, ctx->stream));
    std::vector<double> h((size_t)n * 2 * p);
    for (int c = 0; c < p; ++c)
        for (int i = 0; i < n; ++i) {
            h[(size_t)c * n + i] = B[2 * ((size_t)c * n + i)];
            h[(size_t)(p + c) * n + i] = B[2 * ((size_t)c * n + i) + 1];
        }
    copy_in(ctx, X.d(), N, n, h.data(), n, 2 * p, FL_HOST);
    DBuf Y;
    Y.ensure(sizeof(double) * (size_t)N * P);
    // weight 1: Y = Re(W) for the real RHS; fetch the W planes directly
    filter_apply_dev(f, X.d(), N, 2 * p, Y.d(), N, nullptr, nullptr);
    std::vector<double> wr((size_t)N * P), wi((size_t)N * P);
    CK(cudaMemcpyAsync(wr.data(), f->w_re.p, sizeof(double) * (size_t)N * P, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaMemcpyAsync(wi.data(), f->w_im.p, sizeof(double) * (size_t)N * P, cudaMemcpyDeviceToHost,
                       ctx->stream));
    sync(ctx);
    for (int c = 0; c < p; ++c)
        for (int i = 0; i < n; ++i) {
            const double ar = wr[(size_t)c * N + i], ai = wi[(size_t)c * N + i];
            const double br = wr[(size_t)(p + c) * N + i], bi = wi[(size_t)(p + c) * N + i];
            W[2 * ((size_t)c * n + i)] = ar - bi;
            W[2 * ((size_t)c * n + i) + 1] = ai + br;
        }
}

void node_release(fl_filter* f) {
    auto& pend = f->ctx->pending;
    pend.erase(std::remove(pend.begin(), pend.end(), f), pend.end());
}

}  // namespace

extern "C" {

int fl_node_solve(fl_ctx* ctx, const fl_matrix* A, double zr, double zi, const double* B, int p,
                  double* W, fl_err* err) {
    return guarded(err, [&] {
        if (p < 1) throw Fail{FL_INVALID_ARGUMENT, "node solve: p must be >= 1"};
        CtxLock lk(ctx);
        std::unique_ptr<fl_filter> f = node_filter(ctx, A, zr, zi);
        try {
            node_solve_impl(f.get(), B, p, W);
        } catch (...) {
            node_release(f.get());
            throw;
        }
        node_release(f.get());
    });
}

int fl_node_create(fl_ctx* ctx, const fl_matrix* A, double zr, double zi, int node_index,
                   fl_node** out, fl_err* err) {
    return guarded(err, [&] {
        CtxLock lk(ctx);
        std::unique_ptr<fl_node> nd(new fl_node());
        nd->ctx = ctx;
        nd->node_index = node_index;
        nd->f = node_filter(ctx, A, zr, zi);
        // factor now (a one-column solve rides along), so a singular shift
        // raises here, as the reference constructor does (filterop.cpp:13-23)
        std::vector<double> b(2 * (size_t)A->n, 0.0), w(2 * (size_t)A->n);
        try {
            node_solve_impl(nd->f.get(), b.data(), 1, w.data());
        } catch (Fail& e) {
            node_release(nd->f.get());
            if (e.code == FL_SINGULAR_NODE) {
                char buf[256];
                std::snprintf(buf, sizeof(buf),
                              "factorize_node: singular factorization at node %d (z = %f+%fi)",
                              node_index, zr, zi);
                e.msg = buf;
                e.index = node_index;
            }
            throw;
        } catch (...) {
            node_release(nd->f.get());
            throw;
        }
        ctx_retain(ctx);
        *out = nd.release();
    });
}

int fl_node_factor_solve(fl_node* node, const double* B, int p, double* W, fl_err* err) {
    return guarded(err, [&] {
        if (p < 1) throw Fail{FL_INVALID_ARGUMENT, "node solve: p must be >= 1"};
        CtxLock lk(node->ctx);
        node_solve_impl(node->f.get(), B, p, W);
    });
}

int fl_node_destroy(fl_node* node) {
    if (node) {
        fl_ctx* ctx = node->ctx;
        {
            CtxLock lk(ctx);
            cudaStreamSynchronize(ctx->stream);
            node_release(node->f.get());
            delete node;
        }
        ctx_release(ctx);
    }
    return FL_OK;
}

}  // extern "C"
