// FP64 tensor-core (DMMA) GEMM tiles for sm_100a.
//
// One CTA = 4 warps = a 64x64 output tile; each warp owns 32x32 (4x4 DMMA
// m8n8k4 tiles). Operand tiles (BK = 16 deep) stream global -> shared through
// a cp.async multi-stage ring; fragments are read from padded shared memory
// with conflict-free 8-byte loads:
//   "MK" operand layout (64-dim contiguous in global):  smem[k][x], ld 68
//   "KM" operand layout (k contiguous in global):        smem[x][k ^ 4(x&3)], ld 16
// (the XOR swizzle spreads a fragment read's 8 rows x 4 k over all 16
// 8-byte bank pairs without padding, so a 2-stage planar-complex ring is
// 66 KB and three CTAs fit on one SM).
// Complex operands are planar (separate Re / Im planes), so each DMMA tile is
// purely real; a complex multiply-add is 4 real DMMAs (no 3M trick: keeps the
// rounding of the 4M product the reference's std::complex arithmetic has).
#pragma once
#include "common.cuh"

namespace fl {

constexpr int GB = 64;       // CTA tile (M and N)
constexpr int GK = 16;       // k depth per stage
constexpr int LD_MK = GB + 4;  // 68
constexpr int LD_KM = GK;      // 16, swizzled
constexpr int MK_DOUBLES = GK * LD_MK;  // 1088
constexpr int KM_DOUBLES = GB * LD_KM;  // 1024
constexpr int TILE_DOUBLES = MK_DOUBLES;  // >= either layout

FL_DEV int km_index(int x, int k) { return x * LD_KM + (k ^ ((x & 3) << 2)); }

// Copy one 64x16 operand tile (one plane) into shared memory.
//  KC=false: global column-major with the 64-dim contiguous: tile columns are k.
//  KC=true : global column-major with k contiguous: tile columns are the 64-dim.
template <bool KC, int NT = 128>
FL_DEV void load_tile(double* sm, const double* g, long ld, int tid) {
    if (!KC) {
        // 16 columns x 64 doubles = 16 x 32 chunks of 16 B
#pragma unroll
        for (int i = 0; i < 512 / NT; ++i) {
            int c = tid + i * NT;
            int col = c >> 5, ch = c & 31;
            cp_async16(sm + col * LD_MK + ch * 2, g + col * ld + ch * 2);
        }
    } else {
        // 64 columns x 16 doubles = 64 x 8 chunks
#pragma unroll
        for (int i = 0; i < 512 / NT; ++i) {
            int c = tid + i * NT;
            int col = c >> 3, ch = c & 7;
            cp_async16(sm + km_index(col, ch * 2), g + col * ld + ch * 2);
        }
    }
}

// Fragment element (x, k) of a tile in shared memory.
template <bool KC>
FL_DEV double frag(const double* sm, int x, int k) {
    return KC ? sm[km_index(x, k)] : sm[k * LD_MK + x];
}

// Offset of global tile (x0, k0) for an operand of the given layout.
template <bool KC>
FL_DEV const double* tile_ptr(const double* base, long ld, int x0, int k0) {
    return KC ? base + (long)x0 * ld + k0 : base + (long)k0 * ld + x0;
}

// Tile (bx, by) of the L-th tile of C's lower trapezoid {bx >= by + s},
// column by column (Mt x Nt tiles). Columns c < -s are full (Mt tiles); from
// there column f + j holds H - j tiles, H = Mt - f - s.
FL_DEV void lower_tile(long L, int Mt, int s, int& bx, int& by) {
    const int f = s < 0 ? -s : 0;
    const long full = (long)f * Mt;
    if (L < full) {
        by = (int)(L / Mt);
        bx = (int)(L % Mt);
        return;
    }
    L -= full;
    const long H = (long)Mt - f - s;
    auto cum = [&](long j) { return j * H - j * (j - 1) / 2; };
    const double b = 2.0 * H + 1.0;
    long j = (long)((b - sqrt(fmax(b * b - 8.0 * (double)L, 0.0))) * 0.5);
    if (j < 0) j = 0;
    while (cum(j + 1) <= L) ++j;
    while (j > 0 && cum(j) > L) --j;
    by = (int)(f + j);
    bx = (int)(f + j + s + (L - cum(j)));
}

// Row-group rasterisation of a full Mt x Nt tile grid: CTAs in launch order
// walk groups of R row tiles column by column, so the CTAs in flight share
// R tiles of A's rows (R x K x 16 B stay in L2 for the whole sweep) and
// stream B, instead of sweeping all of A once per tile column (a K = 1024
// L21 panel is ~250 MB per node at cfg4: larger than L2).
FL_DEV void raster_tile(int R, int Mt, int Nt, int& bx, int& by) {
    const long L = (long)by * Mt + bx;
    const long per = (long)R * Nt;
    const int grp = (int)(L / per);
    const int in = (int)(L - (long)grp * per);
    const int rows = min(R, Mt - grp * R);
    by = in / rows;
    bx = grp * R + in - by * rows;
}

}  // namespace fl
