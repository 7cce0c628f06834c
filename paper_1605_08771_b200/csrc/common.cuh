// Shared device helpers for the feastlab B200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define FL_DEV __device__ __forceinline__

// Internal blocking: every device matrix is stored column-major with its row
// count padded to a multiple of FL_TILE (zero rows / identity-free padding, see
// DESIGN.md "Data layout in HBM") so the GEMM-class kernels run without edge
// predication.
#define FL_TILE 64

namespace fl {

// ---------------------------------------------------------------- DMMA
// mma.sync m8n8k4 f64 — one SASS DMMA.8x8x4 (256 FMA). Fragment ownership for
// lane (g = lane>>2, t = lane&3):  a = A[g][t], b = B[t][g],
// c = {C[g][2t], C[g][2t+1]}.
FL_DEV void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// ---------------------------------------------------------------- cp.async
FL_DEV uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
FL_DEV void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem));
}
FL_DEV void cp_async16_zfill(void* smem, const void* gmem, bool valid) {
    int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)),
                 "l"(gmem), "r"(sz));
}
FL_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
FL_DEV void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---------------------------------------------------------------- mbarrier + bulk async copy
FL_DEV void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
FL_DEV void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::); }
FL_DEV void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes));
}
FL_DEV void mbar_wait_parity(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity));
}
// global -> shared bulk copy (the TMA engine), completion counted on `bar`
FL_DEV void bulk_g2s(void* smem, const void* gmem, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(smem)),
        "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// ---------------------------------------------------------------- complex (planar)
struct cplx {
    double re, im;
};
FL_DEV cplx cmul(cplx a, cplx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
FL_DEV cplx crecip(cplx a) {
    // 1/a with Smith's scaling (avoids overflow for large |a|)
    if (fabs(a.re) >= fabs(a.im)) {
        double r = a.im / a.re, d = a.re + a.im * r;
        return {1.0 / d, -r / d};
    } else {
        double r = a.re / a.im, d = a.im + a.re * r;
        return {r / d, -1.0 / d};
    }
}
FL_DEV double cabs2(cplx a) { return a.re * a.re + a.im * a.im; }

// argmax reduction key: larger score wins, ties -> smaller index
FL_DEV bool better(double s1, int i1, double s2, int i2) {
    return (s1 > s2) || (s1 == s2 && i1 < i2);
}

FL_DEV void warp_argmax(double& s, int& idx) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        double so = __shfl_xor_sync(0xffffffffu, s, off);
        int io = __shfl_xor_sync(0xffffffffu, idx, off);
        if (better(so, io, s, idx)) { s = so; idx = io; }
    }
}

FL_DEV double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

}  // namespace fl
