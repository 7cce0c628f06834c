// Latency micro-benchmarks for the panel's column step on B200 (cycles):
// dependent DFMA, double reciprocal, warp argmax level, __syncthreads (256
// threads), cluster barrier (16 CTAs), st.async + mbarrier one-way latency.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_bench tools/lat_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void k_alu(int iters, long long* out, double seed) {
    double x = seed, y = seed * 0.5;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) x = fma(x, 0.999, 1e-3);
    long long t1 = clock64();
    for (int i = 0; i < iters; ++i) y = 1.0 / (y + 1.0);
    long long t2 = clock64();
    double s = x;
    int idx = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        double so = __shfl_xor_sync(0xffffffffu, s, 1 << (i % 5));
        int io = __shfl_xor_sync(0xffffffffu, idx, 1 << (i % 5));
        if (so > s || (so == s && io < idx)) { s = so; idx = io; }
    }
    long long t3 = clock64();
    for (int i = 0; i < iters; ++i) __syncthreads();
    long long t4 = clock64();
    unsigned u = threadIdx.x * 7u;
    for (int i = 0; i < iters; ++i) u = __reduce_max_sync(0xffffffffu, u + threadIdx.x) ^ threadIdx.x;
    long long t5 = clock64();
    double v = seed;
    for (int i = 0; i < iters; ++i) { double w = v * v + 0.5; v = 1.0 / w; }
    long long t6 = clock64();
    if (threadIdx.x == 0) { out[6] = (t5 - t4) / iters; out[7] = (t6 - t5) / iters; out[14] = u + (long long)v; }
    if (threadIdx.x == 0) {
        out[0] = (t1 - t0) / iters;
        out[1] = (t2 - t1) / iters;
        out[2] = (t3 - t2) / iters;
        out[3] = (t4 - t3) / iters;
        out[15] = (long long)(x + y + s + idx);
    }
}

__global__ void __cluster_dims__(8, 1, 1) k_cbar(int iters, long long* out) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[4] = (t1 - t0) / iters;
}

// ping-pong: rank 0 st.async -> rank 1's buffer + mbarrier; rank 1 waits, replies
__global__ void __cluster_dims__(2, 1, 1) k_pingpong(int iters, long long* out) {
    __shared__ __align__(16) double buf[2];
    __shared__ __align__(8) uint64_t bar;
    cg::cluster_group cl = cg::this_cluster();
    const int rank = cl.block_rank();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
    cl.sync();
    const int other = rank ^ 1;
    uint32_t rbuf, rbar;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rbuf) : "r"(su32(buf)), "r"(other));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rbar) : "r"(su32(&bar)), "r"(other));
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int i = 0; i < iters; ++i) {
            const unsigned par = i & 1;
            if (rank == 0) {
                asm volatile(
                    "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(
                        rbuf),
                    "d"(1.0), "d"((double)i), "r"(rbar)
                    : "memory");
            }
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16;\n" ::"r"(su32(&bar)));
            asm volatile(
                "{\n.reg .pred p;\nW_%=:\n"
                "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
                "@!p bra W_%=;\n}\n" ::"r"(su32(&bar)),
                "r"(par)
                : "memory");
            if (rank == 1) {
                asm volatile(
                    "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(
                        rbuf),
                    "d"(1.0), "d"((double)i), "r"(rbar)
                    : "memory");
            }
        }
    }
    long long t1 = clock64();
    cl.sync();
    if (threadIdx.x == 0 && rank == 0) out[5] = (t1 - t0) / iters;  // round trip
}

__device__ __forceinline__ int redux_argmax(unsigned& hi, unsigned& lo, int row) {
    const unsigned m1 = __reduce_max_sync(0xffffffffu, hi);
    const unsigned m2 = __reduce_max_sync(0xffffffffu, hi == m1 ? lo : 0u);
    const unsigned r = __reduce_min_sync(0xffffffffu, (hi == m1 && lo == m2) ? (unsigned)row : 0x7fffffffu);
    hi = m1; lo = m2;
    return m1 == 0u ? 0x7fffffff : (int)r;
}
// candidate phase of the panel column step, isolated: score, reciprocal,
// warp REDUX argmax, winner-row stores, block barrier, CTA REDUX argmax
template <int MODE>  // bit0: reciprocal, bit1: winner-row stores, bit2: CTA stage, bit3: warp REDUX
__global__ void k_cand(int iters, long long* out, double seed) {
    __shared__ double2 wval[2][8][16];
    __shared__ uint4 wkey[2][8];
    __shared__ double2 winv[2][8];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    double2 x[16];
    for (int k = 0; k < 16; ++k) x[k] = make_double2(seed * (tid + 1) * (k + 1) * 1e-3, seed * k);
    int acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int par = it & 1;
        const int jj = it & 15;
        double2 xj = x[0];
#pragma unroll
        for (int k = 0; k < 16; ++k) if (k == jj) xj = x[k];
        const double sc = xj.x * xj.x + xj.y * xj.y;
        const double rs = (MODE & 1) ? 1.0 / ((sc > 0.0 && sc < 1e300) ? sc : 1.0) : sc;
        const double2 myinv = make_double2(xj.x * rs, -xj.y * rs);
        const unsigned long long bits = (unsigned long long)__double_as_longlong(sc);
        unsigned hi = (unsigned)(bits >> 32) + 1u, lo = (unsigned)bits;
        const int wr = (MODE & 8) ? redux_argmax(hi, lo, tid) : (int)(hi & 31);
        if ((MODE & 2) && tid == wr) {
#pragma unroll
            for (int k = 0; k < 16; ++k) wval[par][wid][k] = x[k];
            winv[par][wid] = myinv;
        }
        if (lane == 0) wkey[par][wid] = make_uint4(hi, lo, (unsigned)wr, 0u);
        __syncthreads();
        unsigned chi = 0, clo = 0; int crow = 0x7fffffff;
        if (lane < 8) { const uint4 kk = wkey[par][lane]; chi = kk.x; clo = kk.y; crow = (int)kk.z; }
        if (MODE & 4) crow = redux_argmax(chi, clo, crow);
        acc += crow + (int)wval[par][crow >> 5][jj].x;
        x[0].x += 1e-9 * acc;
    }
    long long t1 = clock64();
    if (tid == 0) { out[8] = (t1 - t0) / iters; out[13] = acc; }
    if (tid == 0) printf("cand MODE %d: %lld cycles\n", MODE, (t1 - t0) / iters);
}

int main() {
    long long* d;
    cudaMalloc(&d, 16 * sizeof(long long));
    cudaMemset(d, 0, 16 * sizeof(long long));
    k_alu<<<1, 256>>>(1000, d, 1.0);
    k_cbar<<<8, 256>>>(1000, d);
    k_pingpong<<<2, 32>>>(1000, d);
        k_cand<0><<<1, 256>>>(1000, d, 1.0);
    k_cand<8><<<1, 256>>>(1000, d, 1.0);
    k_cand<8 | 4><<<1, 256>>>(1000, d, 1.0);
    k_cand<8 | 4 | 2><<<1, 256>>>(1000, d, 1.0);
    k_cand<8 | 4 | 1><<<1, 256>>>(1000, d, 1.0);
    k_cand<15><<<1, 256>>>(1000, d, 1.0);
    k_cand<15><<<1, 32>>>(1000, d, 1.0);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[16];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%s\nDFMA dep %lld | 1/(y+1) dep %lld | argmax level (2 shfl+cmp) %lld | __syncthreads(256) %lld | "
           "cluster barrier(8x256) %lld | st.async ping-pong round trip %lld | REDUX dep %lld | sq+recip dep %lld | candidate phase %lld cycles\n",
           cudaGetErrorString(e), h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8]);
    return 0;
}
