// DMMA GEMM kernels (sm_100a): real C = alpha op(A) op(B) + beta C, and the
// planar-complex update C -= A B used by the LU trailing update and the
// blocked triangular solves of the filter.
#include "gemm.cuh"
#include "kernels.hpp"

#include <cstdlib>
#include <cstring>

namespace fl {

// Number of tiles of that trapezoid (host).
static long lower_tiles(int Mt, int Nt, int s) {
    long t = 0;
    for (int c = 0; c < Nt; ++c) {
        const int lo = c + s > 0 ? c + s : 0;
        if (lo < Mt) t += Mt - lo;
    }
    return t;
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(128) dgemm_kernel(DGemm g) {
    constexpr bool AKC = TA, BKC = !TB;
    constexpr int S = 3;
    extern __shared__ __align__(16) double smem[];
    double* As = smem;                       // S tiles
    double* Bs = smem + S * TILE_DOUBLES;    // S tiles
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gq = lane >> 2, tq = lane & 3;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
    const int m0 = blockIdx.x * GB, n0 = blockIdx.y * GB;
    const long z = blockIdx.z;
    const double* A = g.A + z * g.strideA;
    const double* B = g.B + z * g.strideB;
    double* C = g.C + z * g.strideC;

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const int KT = g.K / GK;
#pragma unroll
    for (int s = 0; s < S - 1; ++s) {
        if (s < KT) {
            load_tile<AKC>(As + s * TILE_DOUBLES, tile_ptr<AKC>(A, g.lda, m0, s * GK), g.lda, tid);
            load_tile<BKC>(Bs + s * TILE_DOUBLES, tile_ptr<BKC>(B, g.ldb, n0, s * GK), g.ldb, tid);
        }
        cp_async_commit();
    }
    for (int kt = 0; kt < KT; ++kt) {
        cp_async_wait<S - 2>();
        __syncthreads();
        const int nk = kt + S - 1;
        if (nk < KT) {
            const int st = nk % S;
            load_tile<AKC>(As + st * TILE_DOUBLES, tile_ptr<AKC>(A, g.lda, m0, nk * GK), g.lda, tid);
            load_tile<BKC>(Bs + st * TILE_DOUBLES, tile_ptr<BKC>(B, g.ldb, n0, nk * GK), g.ldb, tid);
        }
        cp_async_commit();
        const double* as = As + (kt % S) * TILE_DOUBLES;
        const double* bs = Bs + (kt % S) * TILE_DOUBLES;
#pragma unroll
        for (int kk = 0; kk < GK; kk += 4) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = frag<AKC>(as, wm + i * 8 + gq, kk + tq);
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = frag<BKC>(bs, wn + j * 8 + gq, kk + tq);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
        }
    }
    cp_async_wait<0>();
    // epilogue
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = m0 + wm + i * 8 + gq;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = n0 + wn + j * 8 + 2 * tq + e;
                double* cp = C + (long)col * g.ldc + row;
                double v = g.alpha * acc[i][j][e];
                if (g.beta != 0.0) v += g.beta * *cp;
                *cp = v;
            }
        }
    }
}

// Planar complex tile update, A: MxK "MK", B: KxN "KM".
//   SUB: C <- C - A B   (LU trailing update, solve updates). The C tile is
//        loaded straight into the DMMA accumulators before the main loop, so
//        its HBM latency overlaps the first operand tile's cp.async instead of
//        serialising in the epilogue; A fragments are negated in registers.
//   SET: C <- A B       (multiplication by the inverted 64x64 diagonal blocks;
//        in place is safe: a CTA consumes its whole K range before storing).
constexpr int ZSTAGE = 2 * MK_DOUBLES + 2 * KM_DOUBLES;  // Ar Ai Br Bi
constexpr int ZSMEM = 2 * ZSTAGE * sizeof(double);         // 67584 B, 3 CTAs / SM
static_assert(2 * ZSTAGE >= 2 * GB * (GB + 2), "epilogue staging must fit the ring");

#ifndef FL_ZGEMM_MINB
#define FL_ZGEMM_MINB 2
#endif
template <bool SUB>
__global__ void __launch_bounds__(128, FL_ZGEMM_MINB) zgemm_kernel(ZGemm g) {
    extern __shared__ __align__(16) double smem[];
    // per stage: Ar, Ai, Br, Bi
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gq = lane >> 2, tq = lane & 3;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
    int bx = blockIdx.x, by = blockIdx.y;
    if (g.tri) lower_tile(blockIdx.x, g.M / GB, g.tri_s, bx, by);
    const int m0 = bx * GB, n0 = by * GB;
    const long z = blockIdx.z;
    const double* Ar = g.Ar + z * g.strideA;
    const double* Ai = g.Ai + z * g.strideA;
    const double* Br = g.Br + z * g.strideB;
    const double* Bi = g.Bi + z * g.strideB;
    double* Cr = g.Cr + z * g.strideC;
    double* Ci = g.Ci + z * g.strideC;

    auto issue = [&](int st, int kt) {
        double* base = smem + st * ZSTAGE;
        load_tile<false>(base, tile_ptr<false>(Ar, g.lda, m0, kt * GK), g.lda, tid);
        load_tile<false>(base + MK_DOUBLES, tile_ptr<false>(Ai, g.lda, m0, kt * GK), g.lda, tid);
        load_tile<true>(base + 2 * MK_DOUBLES, tile_ptr<true>(Br, g.ldb, n0, kt * GK), g.ldb, tid);
        load_tile<true>(base + 2 * MK_DOUBLES + KM_DOUBLES, tile_ptr<true>(Bi, g.ldb, n0, kt * GK),
                        g.ldb, tid);
    };

    const int KT = g.K / GK;
    if (KT > 0) issue(0, 0);
    cp_async_commit();

    double accr[4][4][2], acci[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                if (SUB) {
                    const long off = (long)(n0 + wn + j * 8 + 2 * tq + e) * g.ldc + m0 + wm + i * 8 + gq;
                    accr[i][j][e] = Cr[off];
                    acci[i][j][e] = Ci[off];
                } else {
                    accr[i][j][e] = 0.0;
                    acci[i][j][e] = 0.0;
                }
            }
    constexpr double sgn = SUB ? -1.0 : 1.0;

    for (int kt = 0; kt < KT; ++kt) {
        cp_async_wait<0>();
        __syncthreads();
        if (kt + 1 < KT) issue((kt + 1) & 1, kt + 1);
        cp_async_commit();
        const double* base = smem + (kt & 1) * ZSTAGE;
        const double* ar_s = base;
        const double* ai_s = base + MK_DOUBLES;
        const double* br_s = base + 2 * MK_DOUBLES;
        const double* bi_s = base + 2 * MK_DOUBLES + KM_DOUBLES;
#pragma unroll
        for (int kk = 0; kk < GK; kk += 4) {
            double ar[4], ai[4], br[4], bi[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                ar[i] = sgn * frag<false>(ar_s, wm + i * 8 + gq, kk + tq);
                ai[i] = sgn * frag<false>(ai_s, wm + i * 8 + gq, kk + tq);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                br[j] = frag<true>(br_s, wn + j * 8 + gq, kk + tq);
                bi[j] = frag<true>(bi_s, wn + j * 8 + gq, kk + tq);
            }
            // four passes over the 16 accumulator tiles: two DMMAs into the
            // same accumulator are 32 instructions apart (no dependent stall);
            // the Im x Im product reuses the Im fragments negated in place
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(accr[i][j], ar[i], br[j]);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acci[i][j], ar[i], bi[j]);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acci[i][j], ai[i], br[j]);
#pragma unroll
            for (int i = 0; i < 4; ++i) ai[i] = -ai[i];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(accr[i][j], ai[i], bi[j]);
        }
        __syncthreads();
    }
    // epilogue staged through the (now free) operand buffers: fragments ->
    // shared memory (ld 66, conflict-free), then fully coalesced 16-byte
    // stores (4 whole 128-byte lines per warp instruction instead of 8-byte
    // scatters over 4 columns): +4-8 % of DMMA peak at K = 64..128
    constexpr int LDC = GB + 2;
    double* sr = smem;
    double* si = smem + GB * LDC;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int o = (wn + j * 8 + 2 * tq + e) * LDC + wm + i * 8 + gq;
                sr[o] = accr[i][j][e];
                si[o] = acci[i][j][e];
            }
    __syncthreads();
    for (int c = tid; c < GB * (GB / 2); c += 128) {
        const int col = c >> 5, ch = c & 31;
        const long off = (long)(n0 + col) * g.ldc + m0 + ch * 2;
        *reinterpret_cast<double2*>(Cr + off) = *reinterpret_cast<const double2*>(sr + col * LDC + ch * 2);
        *reinterpret_cast<double2*>(Ci + off) = *reinterpret_cast<const double2*>(si + col * LDC + ch * 2);
    }
}

// 3M planar complex tile (Gauss/Karatsuba): three real products per k step,
//   T1 = Ar Br,  T2 = Ai Bi,  T3 = (Ar + Ai)(Br + Bi),
//   Re(AB) = T1 - T2,  Im(AB) = T3 - T1 - T2,
// i.e. 3 DMMAs where the 4M form needs 4 (-25 % tensor work). The error is
// normwise (|Im| bounded by eps (|Ar|+|Ai|)(|Br|+|Bi|), Higham, "Stability of
// a method for multiplying complex matrices with three real matrix
// multiplications"), which is what the LU's backward error analysis uses.
// 8 warps, each a 32x16 slice of the 64x64 tile (3 x 16 accumulator
// registers); 3-stage cp.async ring; C is prefetched into L2 when the CTA
// starts and combined in the coalesced epilogue (SUB: C -= AB, SET: C = AB).
template <bool SUB, int NT, int S, int MINB>
__global__ void __launch_bounds__(NT, MINB) zgemm3m_kernel(ZGemm g) {
    constexpr int WN = NT == 256 ? 16 : 32;  // warp tile 32 x WN
    constexpr int NJ = WN / 8;
    extern __shared__ __align__(16) double smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gq = lane >> 2, tq = lane & 3;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * WN;
    int bx = blockIdx.x, by = blockIdx.y;
    if (g.tri) lower_tile(blockIdx.x, g.M / GB, g.tri_s, bx, by);
    else if (g.raster > 0) raster_tile(g.raster, g.M / GB, g.N / GB, bx, by);
    const int m0 = bx * GB, n0 = by * GB;
    const long z = blockIdx.z;
    const double* Ar = g.Ar + z * g.strideA;
    const double* Ai = g.Ai + z * g.strideA;
    const double* Br = g.Br + z * g.strideB;
    const double* Bi = g.Bi + z * g.strideB;
    double* Cr = g.Cr + z * g.strideC;
    double* Ci = g.Ci + z * g.strideC;

    if (SUB && tid < 2 * GB) {  // one 512-byte column segment per thread
        const double* c = (tid < GB ? Cr : Ci) + (long)(n0 + (tid & (GB - 1))) * g.ldc + m0;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], 512;\n" ::"l"(c) : "memory");
    }

    auto issue = [&](int st, int kt) {
        double* base = smem + st * ZSTAGE;
        load_tile<false, NT>(base, tile_ptr<false>(Ar, g.lda, m0, kt * GK), g.lda, tid);
        load_tile<false, NT>(base + MK_DOUBLES, tile_ptr<false>(Ai, g.lda, m0, kt * GK), g.lda, tid);
        load_tile<true, NT>(base + 2 * MK_DOUBLES, tile_ptr<true>(Br, g.ldb, n0, kt * GK), g.ldb,
                             tid);
        load_tile<true, NT>(base + 2 * MK_DOUBLES + KM_DOUBLES,
                             tile_ptr<true>(Bi, g.ldb, n0, kt * GK), g.ldb, tid);
    };

    const int KT = g.K / GK;
#pragma unroll
    for (int s = 0; s < S - 1; ++s) {
        if (s < KT) issue(s, s);
        cp_async_commit();
    }
    double t1[4][NJ][2], t2[4][NJ][2], t3[4][NJ][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) t1[i][j][e] = t2[i][j][e] = t3[i][j][e] = 0.0;

    for (int kt = 0; kt < KT; ++kt) {
        cp_async_wait<S - 2>();
        __syncthreads();
        if (kt + S - 1 < KT) issue((kt + S - 1) % S, kt + S - 1);
        cp_async_commit();
        const double* base = smem + (kt % S) * ZSTAGE;
        const double* ar_s = base;
        const double* ai_s = base + MK_DOUBLES;
        const double* br_s = base + 2 * MK_DOUBLES;
        const double* bi_s = base + 2 * MK_DOUBLES + KM_DOUBLES;
#pragma unroll
        for (int kk = 0; kk < GK; kk += 4) {
            double ar[4], ai[4], as[4], br[NJ], bi[NJ], bs[NJ];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                ar[i] = frag<false>(ar_s, wm + i * 8 + gq, kk + tq);
                ai[i] = frag<false>(ai_s, wm + i * 8 + gq, kk + tq);
                as[i] = ar[i] + ai[i];
            }
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                br[j] = frag<true>(br_s, wn + j * 8 + gq, kk + tq);
                bi[j] = frag<true>(bi_s, wn + j * 8 + gq, kk + tq);
                bs[j] = br[j] + bi[j];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < NJ; ++j) dmma(t1[i][j], ar[i], br[j]);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < NJ; ++j) dmma(t2[i][j], ai[i], bi[j]);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < NJ; ++j) dmma(t3[i][j], as[i], bs[j]);
        }
    }
    cp_async_wait<0>();
    __syncthreads();
    constexpr int LDC = GB + 2;
    double* sr = smem;
    double* si = smem + GB * LDC;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int o = (wn + j * 8 + 2 * tq + e) * LDC + wm + i * 8 + gq;
                sr[o] = t1[i][j][e] - t2[i][j][e];
                si[o] = t3[i][j][e] - t1[i][j][e] - t2[i][j][e];
            }
    __syncthreads();
#pragma unroll
    for (int c = tid; c < GB * (GB / 2); c += NT) {
        const int col = c >> 5, ch = c & 31;
        const long off = (long)(n0 + col) * g.ldc + m0 + ch * 2;
        double2 dr = *reinterpret_cast<const double2*>(sr + col * LDC + ch * 2);
        double2 di = *reinterpret_cast<const double2*>(si + col * LDC + ch * 2);
        if (SUB) {
            const double2 cr = *reinterpret_cast<const double2*>(Cr + off);
            const double2 ci = *reinterpret_cast<const double2*>(Ci + off);
            dr = make_double2(cr.x - dr.x, cr.y - dr.y);
            di = make_double2(ci.x - di.x, ci.y - di.y);
        }
        *reinterpret_cast<double2*>(Cr + off) = dr;
        *reinterpret_cast<double2*>(Ci + off) = di;
    }
}

// 3M launch shapes: 4 warps of 32x32 (242 registers, 2 CTAs / SM) stream
// the long-K updates best; 8 warps of 32x16 (2 CTAs of 256 threads) hide
// the prologue / epilogue of short-K (64) products better.
template <bool SUB>
void launch_zgemm3m(const ZGemm& g, dim3 grid, cudaStream_t s) {
    constexpr int smem = 3 * ZSTAGE * sizeof(double);
    if (g.K >= 128) {
        ensure_smem((const void*)zgemm3m_kernel<SUB, 128, 3, 2>, smem);
        zgemm3m_kernel<SUB, 128, 3, 2><<<grid, 128, smem, s>>>(g);
    } else {
        ensure_smem((const void*)zgemm3m_kernel<SUB, 256, 3, 2>, smem);
        zgemm3m_kernel<SUB, 256, 3, 2><<<grid, 256, smem, s>>>(g);
    }
}

static int g_zgemm_mode = -1;  // 0 = 4M, 1 = 3M; -1 = from FEASTLAB_ZGEMM (default 3m)

int zgemm_mode() {
    if (g_zgemm_mode < 0) {
        const char* e = std::getenv("FEASTLAB_ZGEMM");
        g_zgemm_mode = (e && std::strcmp(e, "4m") == 0) ? 0 : 1;
    }
    return g_zgemm_mode;
}
void set_zgemm_mode(int mode) { g_zgemm_mode = mode ? 1 : 0; }

void launch_dgemm(const DGemm& g, bool ta, bool tb, int batch, cudaStream_t s) {
    if (g.M <= 0 || g.N <= 0 || batch <= 0) return;
    dim3 grid(g.M / GB, g.N / GB, batch);
    const size_t sm = 3 * 2 * TILE_DOUBLES * sizeof(double);
#define FL_DG(TA, TB)                                                                        \
    {                                                                                        \
        ensure_smem((const void*)dgemm_kernel<TA, TB>, sm);                                  \
        dgemm_kernel<TA, TB><<<grid, 128, sm, s>>>(g);                                       \
    }
    if (!ta && !tb) FL_DG(false, false)
    else if (ta && !tb) FL_DG(true, false)
    else if (!ta && tb) FL_DG(false, true)
    else FL_DG(true, true)
#undef FL_DG
}

// Row tiles per raster group (FEASTLAB_ZGEMM_RASTER, 0 = column-major launch order)
static int raster_rows() {
    static const int r = [] {
        const char* e = std::getenv("FEASTLAB_ZGEMM_RASTER");
        return e ? std::atoi(e) : 0;
    }();
    return r;
}

void launch_zgemm_sub(const ZGemm& g0, int batch, cudaStream_t s) {
    if (g0.M <= 0 || g0.N <= 0 || g0.K <= 0 || batch <= 0) return;
    ZGemm g = g0;
    dim3 grid(g.M / GB, g.N / GB, batch);
    if (zgemm_mode()) {
        // only where a tile column does not already fit: several tile columns
        if (g.N / GB > 1 && g.M / GB > raster_rows()) g.raster = raster_rows();
        launch_zgemm3m<true>(g, grid, s);
        return;
    }
    const size_t sm = ZSMEM;
    ensure_smem((const void*)zgemm_kernel<true>, sm);
    zgemm_kernel<true><<<grid, 128, sm, s>>>(g);
}

void launch_zgemm_sub_lower(const ZGemm& g0, int tri_s, int batch, cudaStream_t s) {
    if (g0.M <= 0 || g0.N <= 0 || g0.K <= 0 || batch <= 0) return;
    ZGemm g = g0;
    g.tri = true;
    g.tri_s = tri_s;
    const long t = lower_tiles(g.M / GB, g.N / GB, tri_s);
    if (t <= 0) return;
    dim3 grid((unsigned)t, 1, batch);
    if (zgemm_mode()) {
        launch_zgemm3m<true>(g, grid, s);
        return;
    }
    const size_t sm = ZSMEM;
    ensure_smem((const void*)zgemm_kernel<true>, sm);
    zgemm_kernel<true><<<grid, 128, sm, s>>>(g);
}

void launch_zgemm_set(const ZGemm& g, int batch, cudaStream_t s) {
    if (g.M <= 0 || g.N <= 0 || batch <= 0) return;
    dim3 grid(g.M / GB, g.N / GB, batch);
    if (zgemm_mode()) {
        launch_zgemm3m<false>(g, grid, s);
        return;
    }
    const size_t sm = ZSMEM;
    ensure_smem((const void*)zgemm_kernel<false>, sm);
    zgemm_kernel<false><<<grid, 128, sm, s>>>(g);
}

}  // namespace fl
