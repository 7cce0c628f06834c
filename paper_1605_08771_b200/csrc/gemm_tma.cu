// TMA-fed 3M planar-complex DMMA GEMM for the long-K trailing updates
// (C -= A B with A = L21, B = U12 of an LU / LDL^T outer block; SURVEY.md
// §8(a) a8, north_star "FP64 tensor-core tiles fed by TMA").
//
// Differences from zgemm3m_kernel (gemm.cu):
//  * every operand tile arrives by cp.async.bulk.tensor (one elected thread,
//    mbarrier full/empty ring of 4 stages x 8 k, loads 3 tiles ahead): no
//    LDGSTS, no per-thread address arithmetic, no CTA-wide barrier in the main
//    loop -- the four warps of a CTA drift apart instead of meeting at a
//    __syncthreads every k-tile;
//  * the third product's operands As = Ar + Ai, Bs = Br + Bi are read as
//    precomputed planes (zsum_kernel writes them once per outer block, the
//    same rounded sums the DADDs formed in registers) instead of being summed
//    per fragment: a DADD that depends on a fresh LDS costs the DMMA pipe
//    ~6 % (tools/dmma_mix.cu: 16 LDS + 8 DADD per 48 DMMA 34.99 TF/s, 24 LDS
//    and no DADD 37.00 of 37.1);
//  * shared-memory tiles are dense and hardware-swizzled (SWIZZLE_128B for
//    the 64-contiguous operand, loaded as one 4-D box {16 m, 8 k, 4 m-groups};
//    SWIZZLE_64B for the k-contiguous one), and the k index each DMMA lane
//    reads is permuted ({0,3,4,7} then {1,2,5,6} of a tile's 8) so that all
//    fragment loads are bank-conflict free under both swizzles.
#include <cuda.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "gemm.cuh"
#include "kernels.hpp"

namespace fl {

namespace {

constexpr int TK = 8;                         // k per stage
constexpr int TS = 4;                         // stages
constexpr int LEAD = 3;                       // tile kt + LEAD is issued in the middle of tile kt
constexpr int PLANE_B = GB * TK * 8;          // 4096 B: one 64 x 8 plane
constexpr int STAGE_B = 6 * PLANE_B;          // Ar Ai As Br Bi Bs
constexpr int TMA_SMEM = TS * STAGE_B + 1024 /* alignment slack */ + 64 /* barriers */;
static_assert(TS * STAGE_B >= 2 * GB * (GB + 2) * 8, "epilogue staging must fit the ring");

FL_DEV void tma_load_4d(void* smem, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                        uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(smem_u32(smem)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}
FL_DEV void tma_load_3d(void* smem, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(smem)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
FL_DEV void mbar_arrive_release(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// wait with a compiler memory barrier: the fragment loads are plain C++ loads
// and must not be hoisted above the wait for their tile
FL_DEV void mbar_wait_acquire(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

}  // namespace

// C tile (bx, by) -= sum over K of A B, 3M form with precomputed sum planes.
template <bool SUB>
__global__ void __launch_bounds__(128, 2)
    zgemm3s_kernel(const __grid_constant__ CUtensorMap mAr, const __grid_constant__ CUtensorMap mAi,
                   const __grid_constant__ CUtensorMap mAs, const __grid_constant__ CUtensorMap mBr,
                   const __grid_constant__ CUtensorMap mBi, const __grid_constant__ CUtensorMap mBs,
                   ZGemmTma g) {
    extern __shared__ unsigned char smem_raw[];
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;  // SWIZZLE_128B atoms
    unsigned char* tiles = smem_raw + (base - smem_u32(smem_raw));
    uint64_t* full = reinterpret_cast<uint64_t*>(tiles + TS * STAGE_B);
    uint64_t* empty = full + TS;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gq = lane >> 2, tq = lane & 3;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;
    int bx = blockIdx.x, by = blockIdx.y;
    if (g.tri) lower_tile(blockIdx.x, g.M / GB, g.tri_s, bx, by);
    else if (g.raster > 0) raster_tile(g.raster, g.M / GB, g.N / GB, bx, by);
    const int m0 = bx * GB, n0 = by * GB;
    const int z = blockIdx.z;
    double* Cr = g.Cr + (long)z * g.strideC;
    double* Ci = g.Ci + (long)z * g.strideC;

    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < TS; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 4);
        }
        mbar_fence_init();
    }
    __syncthreads();
    // the C tile is pulled into L2 a few tiles before the epilogue reads it (a
    // prefetch at CTA start is evicted again over a K = 1024 main loop)
    auto prefetch_c = [&] {
        if (SUB && tid < 2 * GB) {  // one 512-byte column segment of the C tile per thread
            const double* c = (tid < GB ? Cr : Ci) + (long)(n0 + (tid & (GB - 1))) * g.ldc + m0;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], 512;\n" ::"l"(c) : "memory");
        }
    };

    const int KT = g.K / TK;
    const int kt_c = KT > 12 ? KT - 12 : 0;  // tile at which the C prefetch is issued
    // tile kt -> stage kt % TS: six boxes, 24 KB, one mbarrier transaction
    auto produce = [&](int kt) {
        const int s = kt % TS;
        if (kt >= TS) mbar_wait_parity(empty + s, ((kt / TS) - 1) & 1);
        unsigned char* st = tiles + s * STAGE_B;
        mbar_arrive_expect_tx(full + s, STAGE_B);
        const int k = kt * TK;
        tma_load_4d(st, &mAr, 0, g.a_col + k, (g.a_row + m0) >> 4, g.a_node + z, full + s);
        tma_load_4d(st + PLANE_B, &mAi, 0, g.a_col + k, (g.a_row + m0) >> 4, g.a_node + z, full + s);
        tma_load_4d(st + 2 * PLANE_B, &mAs, 0, g.as_col + k, (g.as_row + m0) >> 4, g.as_node + z,
                    full + s);
        tma_load_3d(st + 3 * PLANE_B, &mBr, g.b_row + k, g.b_col + n0, g.b_node + z, full + s);
        tma_load_3d(st + 4 * PLANE_B, &mBi, g.b_row + k, g.b_col + n0, g.b_node + z, full + s);
        tma_load_3d(st + 5 * PLANE_B, &mBs, g.bs_row + k, g.bs_col + n0, g.bs_node + z, full + s);
    };
    if (tid == 0) {
#pragma unroll
        for (int d = 0; d < LEAD; ++d)
            if (d < KT) produce(d);
    }

    // Lane offsets inside a stage. DMMA step c (0, 1) of a tile reads
    // k = KSEL[tq] ^ c, KSEL = {0, 3, 4, 7}.
    //  A plane (box {16 mi, 8 k, 4 mo}, SWIZZLE_128B): byte = mo*1024 + k*128 +
    //    ((mi/2) ^ k) * 16 + (mi & 1) * 8, row m = 16 mo + mi = wm + 8 i + gq.
    //  B plane (box {8 k, 64 n}, SWIZZLE_64B): byte = n*64 + (((k/2) ^ (n/2)) & 3) * 16
    //    + (k & 1) * 8, column n = wn + 8 j + gq.
    const int ksel = ((tq & 1) * 3) | ((tq >> 1) << 2);  // 0, 3, 4, 7
    uint32_t offA[2][2];  // [c][i & 1]; add (wm/16 + i/2) * 1024
    uint32_t offB[2];     // [c]; add j * 512
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const int k = ksel ^ c;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int mi = 8 * h + gq;
            offA[c][h] = (wm >> 4) * 1024 + k * 128 + (((mi >> 1) ^ k) << 4) + ((mi & 1) << 3);
        }
        const int n = wn + gq;
        offB[c] = n * 64 + ((((k >> 1) ^ (n >> 1)) & 3) << 4) + ((k & 1) << 3);
    }

    double t1[4][4][2], t2[4][4][2], t3[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) t1[i][j][e] = t2[i][j][e] = t3[i][j][e] = 0.0;

    // Main loop. The fragment loads are plain shared-memory loads, so ptxas
    // interleaves the next k-step's with the current DMMAs as registers free up
    // (192 accumulator + 48 fragment registers); the waits and releases are
    // compiler memory barriers. Tile kt + LEAD reuses the stage of tile kt - 1,
    // which the other warps have left by the middle of tile kt: the producer
    // thread issues it there and rarely blocks.
    // unrolled by the ring depth: stage addresses, barrier addresses and the
    // producing warp become compile-time per copy (0.937 -> 0.954 of the DMMA
    // issue peak; a CTA alone on its SM 0.72 -> 0.76)
#pragma unroll 4
    for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % TS;
        if (kt == kt_c) prefetch_c();
        mbar_wait_acquire(full + s, (kt / TS) & 1);
        const unsigned char* st = tiles + s * STAGE_B;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            // The producer role rotates over the four warps (tile t is issued by
            // lane 0 of warp t & 3): both CTAs of an SM keep their warp w on
            // sub-partition w, so a fixed producer warp would put all the TMA
            // issue work of the SM on one sub-partition (FEASTLAB_TMA_ROTATE=0).
            if (c == 1 && lane == 0 && warp == (g.rotate ? ((kt + LEAD) & 3) : 0) && kt + LEAD < KT)
                produce(kt + LEAD);
            double ar[4], ai[4], as[4], br[4], bi[4], bs[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const unsigned char* a = st + offA[c][i & 1] + (i >> 1) * 1024;
                ar[i] = *reinterpret_cast<const double*>(a);
                ai[i] = *reinterpret_cast<const double*>(a + PLANE_B);
                as[i] = *reinterpret_cast<const double*>(a + 2 * PLANE_B);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const unsigned char* b = st + 3 * PLANE_B + offB[c] + j * 512;
                br[j] = *reinterpret_cast<const double*>(b);
                bi[j] = *reinterpret_cast<const double*>(b + PLANE_B);
                bs[j] = *reinterpret_cast<const double*>(b + 2 * PLANE_B);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(t1[i][j], ar[i], br[j]);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(t2[i][j], ai[i], bi[j]);
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(t3[i][j], as[i], bs[j]);
        }
        // The stage goes back to the TMA engine: a cross-proxy fence orders this
        // warp's generic-proxy reads of it before the async-proxy writes that
        // follow the release. Without it single C tiles came out wrong (about one
        // CTA in 10^6), and only when the look-ahead panel chain ran beside the
        // update and skewed the warps of a CTA against each other.
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive_release(empty + s);
    }
    __syncthreads();  // every warp has read its last tile: the ring becomes the staging buffer
    constexpr int LDC = GB + 2;
    double* sr = reinterpret_cast<double*>(tiles);
    double* si = sr + GB * LDC;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int o = (wn + j * 8 + 2 * tq + e) * LDC + wm + i * 8 + gq;
                sr[o] = t1[i][j][e] - t2[i][j][e];
                si[o] = t3[i][j][e] - t1[i][j][e] - t2[i][j][e];
            }
    // the whole C tile in flight at once (the accumulator registers are free
    // now): one DRAM / L2 round trip per CTA instead of one per 128-byte row
    double2 cr[16], ci[16];
    if (SUB) {
#pragma unroll
        for (int it = 0; it < 16; ++it) {
            const int c = tid + it * 128, col = c >> 5, ch = c & 31;
            const long off = (long)(n0 + col) * g.ldc + m0 + ch * 2;
            cr[it] = *reinterpret_cast<const double2*>(Cr + off);
            ci[it] = *reinterpret_cast<const double2*>(Ci + off);
        }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < 16; ++it) {
        const int c = tid + it * 128, col = c >> 5, ch = c & 31;
        const long off = (long)(n0 + col) * g.ldc + m0 + ch * 2;
        double2 dr = *reinterpret_cast<const double2*>(sr + col * LDC + ch * 2);
        double2 di = *reinterpret_cast<const double2*>(si + col * LDC + ch * 2);
        if (SUB) {
            dr = make_double2(cr[it].x - dr.x, cr[it].y - dr.y);
            di = make_double2(ci[it].x - di.x, ci[it].y - di.y);
        }
        *reinterpret_cast<double2*>(Cr + off) = dr;
        *reinterpret_cast<double2*>(Ci + off) = di;
    }
}

// S = Re + Im over a rows x cols block (both planes ld `ld`), into a plane of
// leading dimension lds: the 3M product's third operand, rounded exactly as
// the in-register DADD of zgemm3m_kernel rounds it.
__global__ void __launch_bounds__(256) zsum_kernel(const double* __restrict__ re,
                                                   const double* __restrict__ im, long ld,
                                                   long stride, double* __restrict__ out, long lds,
                                                   long ostride, int rows, int cols) {
    const int r = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
    const int c = blockIdx.y;
    if (r >= rows) return;
    const long b = blockIdx.z;
    const double2 a = *reinterpret_cast<const double2*>(re + b * stride + (long)c * ld + r);
    const double2 i = *reinterpret_cast<const double2*>(im + b * stride + (long)c * ld + r);
    *reinterpret_cast<double2*>(out + b * ostride + (long)c * lds + r) =
        make_double2(a.x + i.x, a.y + i.y);
}

void launch_zsum(const double* re, const double* im, long ld, long stride, double* out, long lds,
                 long ostride, int rows, int cols, int batch, cudaStream_t s) {
    if (rows <= 0 || cols <= 0 || batch <= 0) return;
    dim3 grid((rows / 2 + 255) / 256, cols, batch);
    zsum_kernel<<<grid, 256, 0, s>>>(re, im, ld, stride, out, lds, ostride, rows, cols);
}

// ------------------------------------------------------------------ tensor maps
namespace {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeFn>(p);
    }();
    if (!fn) throw LaunchError("cuTensorMapEncodeTiled is not available from this driver");
    return fn;
}

}  // namespace

// The 64-contiguous ("MK") operand view of `batch` column-major planes
// (rows x cols, ld, `stride` doubles apart): 4-D {16 mi, cols, rows/16 mo, batch}
// with box {16, 8, 4, 1} -> shared memory [mo][k][mi], SWIZZLE_128B.
void make_tma_map_mk(CUtensorMap* m, const double* base, long rows, long cols, long ld, long stride,
                     int batch) {
    const cuuint64_t dims[4] = {16, (cuuint64_t)cols, (cuuint64_t)(rows / 16), (cuuint64_t)batch};
    const cuuint64_t strides[3] = {(cuuint64_t)ld * 8, 128, (cuuint64_t)stride * 8};
    const cuuint32_t box[4] = {16, TK, 4, 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base),
                                   dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw LaunchError("cuTensorMapEncodeTiled(MK operand) failed: " + std::to_string((int)r));
}

// The k-contiguous ("KM") operand view: 3-D {rows (k), cols, batch}, box
// {8, 64, 1} -> shared memory [n][k], SWIZZLE_64B.
void make_tma_map_km(CUtensorMap* m, const double* base, long rows, long cols, long ld, long stride,
                     int batch) {
    const cuuint64_t dims[3] = {(cuuint64_t)rows, (cuuint64_t)cols, (cuuint64_t)batch};
    const cuuint64_t strides[2] = {(cuuint64_t)ld * 8, (cuuint64_t)stride * 8};
    const cuuint32_t box[3] = {TK, GB, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base),
                                   dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw LaunchError("cuTensorMapEncodeTiled(KM operand) failed: " + std::to_string((int)r));
}

static int tma_raster_rows() {
    static const int r = [] {
        const char* e = std::getenv("FEASTLAB_ZGEMM_RASTER");
        return e ? std::atoi(e) : 16;
    }();
    return r;
}

void launch_zgemm_sub_tma(const ZGemmMaps& m, const ZGemmTma& g0, int batch, cudaStream_t s) {
    if (g0.M <= 0 || g0.N <= 0 || g0.K <= 0 || batch <= 0) return;
    if (g0.M % GB || g0.N % GB || g0.K % TK) throw LaunchError("launch_zgemm_sub_tma: bad shape");
    ZGemmTma g = g0;
    dim3 grid(g.M / GB, g.N / GB, batch);
    if (g.tri) {
        long t = 0;
        for (int c = 0; c < g.N / GB; ++c) {
            const int lo = c + g.tri_s > 0 ? c + g.tri_s : 0;
            if (lo < g.M / GB) t += g.M / GB - lo;
        }
        if (t <= 0) return;
        grid = dim3((unsigned)t, 1, batch);
    } else if (g.N / GB > 1 && g.M / GB > tma_raster_rows()) {
        g.raster = tma_raster_rows();
    }
    static const int rotate = [] {
        const char* e = std::getenv("FEASTLAB_TMA_ROTATE");
        return e ? std::atoi(e) : 1;
    }();
    g.rotate = rotate;
    ensure_smem((const void*)zgemm3s_kernel<true>, TMA_SMEM);
    zgemm3s_kernel<true><<<grid, 128, TMA_SMEM, s>>>(m.Ar, m.Ai, m.As, m.Br, m.Bi, m.Bs, g);
}

}  // namespace fl
