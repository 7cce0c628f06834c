// micro-benchmark: cluster barrier / DSMEM / __syncthreads latencies on B200
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void __cluster_dims__(8,1,1) k_cs(int iters, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (t1 - t0) / iters;
}
__global__ void __cluster_dims__(8,1,1) k_cs_arrive(int iters, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (t1 - t0) / iters;
}
__global__ void k_st(int iters, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[2] = (t1 - t0) / iters;
}
__global__ void __cluster_dims__(8,1,1) k_dsmem(int iters, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ volatile double v[32];
  if (threadIdx.x < 32) v[threadIdx.x] = threadIdx.x;
  cl.sync();
  double acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    volatile double* r = cl.map_shared_rank((double*)v, (i + 1) & 7);
    acc += r[(int)acc & 31];
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[3] = (t1 - t0) / iters; out[7] = (long long)acc; }
  cl.sync();
}
int main() {
  long long* d; cudaMalloc(&d, 64); long long h[8] = {0};
  for (int threads : {256, 512}) {
    k_cs<<<8, threads>>>(1000, d); k_cs_arrive<<<8, threads>>>(1000, d); k_st<<<1, threads>>>(1000, d);
    k_dsmem<<<8, threads>>>(1000, d);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    printf("threads=%d cluster.sync=%lld relaxed arrive/wait=%lld __syncthreads=%lld dsmem_dep_load=%lld cycles (%s)\n",
           threads, h[0], h[1], h[2], h[3], cudaGetErrorString(cudaGetLastError()));
  }
}
