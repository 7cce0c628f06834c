// FP64 peak micro-benchmark for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64) and DFMA.
// Prints one JSON line: {"dmma_tflops":..,"dfma_tflops":..,"sm_count":..,"clock_mhz":..}
#include <cstdio>
#include <cuda_runtime.h>

template <int ITERS>
__global__ void dmma_loop(double* out, double seed) {
    double a = seed + threadIdx.x, b = seed * 0.5 + threadIdx.x;
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 1234.5) out[threadIdx.x] = s;
}

template <int ITERS>
__global__ void dfma_loop(double* out, double seed) {
    double a = seed + threadIdx.x, b = seed * 0.5;
    double c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i] = fma(a, c[i], b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i];
    if (s == 1234.5) out[threadIdx.x] = s;
}

int main() {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    int sms = prop.multiProcessorCount;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* out;
    cudaMalloc(&out, 4096 * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int ITERS = 4096;
    double best_dmma = 0, best_dfma = 0;
    for (int threads : {128, 256, 512}) {
        for (int bps : {1, 2, 4}) {
            int blocks = sms * bps;
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(e0);
                dmma_loop<ITERS><<<blocks, threads>>>(out, 1.0);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                double flops = 2.0 * 256 * 8 * (double)ITERS * blocks * (threads / 32);
                double tf = flops / (ms * 1e-3) / 1e12;
                if (tf > best_dmma) best_dmma = tf;
                cudaEventRecord(e0);
                dfma_loop<ITERS><<<blocks, threads>>>(out, 1.0);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
                flops = 2.0 * 8 * (double)ITERS * blocks * threads;
                tf = flops / (ms * 1e-3) / 1e12;
                if (tf > best_dfma) best_dfma = tf;
            }
        }
    }
    // sustained: long DMMA run (~2 s)
    float total = 0;
    double sflops = 0;
    for (int rep = 0; rep < 40; ++rep) {
        cudaEventRecord(e0);
        dmma_loop<ITERS * 8><<<sms * 2, 256>>>(out, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        total += ms;
        sflops += 2.0 * 256 * 8 * (double)ITERS * 8 * sms * 2 * 8;
    }
    double sustained = sflops / (total * 1e-3) / 1e12;
    printf("{\"dmma_tflops_burst\": %.3f, \"dfma_tflops_burst\": %.3f, \"dmma_tflops_sustained\": %.3f, "
           "\"sm_count\": %d, \"clock_mhz_attr\": %d, \"err\": \"%s\"}\n",
           best_dmma, best_dfma, sustained, sms, clk / 1000, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
