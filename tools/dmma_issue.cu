// DMMA issue micro-benchmark (sm_100a): how many warps per SM sub-partition,
// and how many independent accumulators per warp, does the FP64 tensor pipe
// need to run at its peak?  One JSON line per (threads, CTAs/SM, ILP).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_issue tools/dmma_issue.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP, bool LDS>
__global__ void loop(double* out, double seed, int iters) {
    __shared__ double sm[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = seed + i;
    __syncthreads();
    double a = seed + threadIdx.x, b = seed * 0.5 + threadIdx.x;
    double c[ILP][2];
#pragma unroll
    for (int i = 0; i < ILP; ++i) c[i][0] = c[i][1] = 0;
    const int lane = threadIdx.x & 31;
    for (int it = 0; it < iters; ++it) {
        if (LDS) {  // the zgemm3m ratio: 16 fragment loads + 8 DADD per 48 DMMAs
            double f[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) f[k] = sm[((it + k) * 32 + lane) & 2047];
#pragma unroll
            for (int k = 0; k < 8; ++k) f[k] += f[k + 8];
#pragma unroll
            for (int i = 0; i < ILP; ++i)
                asm volatile(
                    "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                    : "+d"(c[i][0]), "+d"(c[i][1])
                    : "d"(f[i & 7]), "d"(f[8 + (i & 7)]));
        } else {
#pragma unroll
            for (int i = 0; i < ILP; ++i)
                asm volatile(
                    "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                    : "+d"(c[i][0]), "+d"(c[i][1])
                    : "d"(a), "d"(b));
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1];
    if (s == 1234.5) out[threadIdx.x] = s;
}

template <int ILP, bool LDS>
void run(double* out, int sms, int threads, int bps) {
    const int iters = 4096 * 8 / ILP;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        loop<ILP, LDS><<<sms * bps, threads>>>(out, 1.0, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * 256 * ILP * (double)iters * sms * bps * (threads / 32);
    printf("{\"threads\": %d, \"ctas_per_sm\": %d, \"warps_per_smsp\": %.1f, \"ilp\": %d, \"lds\": %d, "
           "\"tflops\": %.2f}\n",
           threads, bps, threads / 32 * bps / 4.0, ILP, (int)LDS, flops / (best * 1e-3) / 1e12);
}

int main() {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    const int sms = prop.multiProcessorCount;
    double* out;
    cudaMalloc(&out, 4096 * sizeof(double));
    const int cfg[][2] = {{128, 1}, {128, 2}, {128, 3}, {128, 4}, {256, 1}, {256, 2}, {512, 1}};
    for (auto& c : cfg) {
        run<1, false>(out, sms, c[0], c[1]);
        run<2, false>(out, sms, c[0], c[1]);
        run<4, false>(out, sms, c[0], c[1]);
        run<8, false>(out, sms, c[0], c[1]);
        run<16, false>(out, sms, c[0], c[1]);
        run<48, false>(out, sms, c[0], c[1]);
        run<48, true>(out, sms, c[0], c[1]);
    }
    printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
