// time fl::jacobi_eig (device symmetric eigensolver) per sweep on random matrices
#include <cstdio>
#include <vector>
#include <random>
#include <cuda_runtime.h>
#include "../paper_1605_08771_b200/csrc/ritz_kernels.hpp"
int main() {
  for (int p : {150, 400, 768, 1320}) {
    const int P = (p + 63) / 64 * 64;
    std::vector<double> h((size_t)P * P, 0.0);
    std::mt19937_64 g(1); std::normal_distribution<double> nd;
    for (int j = 0; j < p; ++j) for (int i = 0; i <= j; ++i) { double v = nd(g); h[(size_t)j * P + i] = v; h[(size_t)i * P + j] = v; }
    double fro = 0; for (double v : h) fro += v * v; fro = sqrt(fro);
    double *A, *W, *V, *Vo, *vals; int* si; unsigned long long* cnt;
    cudaMalloc(&A, 8ul * P * P); cudaMalloc(&W, 8ul * P * P); cudaMalloc(&V, 8ul * P * P); cudaMalloc(&Vo, 8ul * P * P);
    cudaMalloc(&vals, 8ul * P); cudaMalloc(&si, 64); cudaMalloc(&cnt, 8 * 64);
    for (int sweeps : {1, 40}) {
      cudaMemcpy(A, h.data(), 8ul * P * P, cudaMemcpyHostToDevice);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      int rc = fl::jacobi_eig(A, P, p, fro, W, V, P, vals, Vo, P, si, cnt, sweeps, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      int done = 0; cudaMemcpy(&done, si, 4, cudaMemcpyDeviceToHost);
      printf("p=%d max_sweeps=%d: %.2f ms, sweeps %d, %.2f us/round rc=%d %s\n", p, sweeps, ms, done,
             1000.0 * ms / (done * (p + (p & 1) - 1)), rc, cudaGetErrorString(cudaGetLastError()));
    }
  }
}
