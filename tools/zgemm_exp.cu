// Experiment: where does the short-K DMMA GEMM lose time? Variants of the
// one-tile-per-CTA planar complex kernel with C load / C store switched off,
// and with the epilogue staged through shared memory (coalesced 16-B stores).
#include <cstdio>
#include <cuda_runtime.h>
#define DEV __device__ __forceinline__
DEV void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
DEV unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
DEV void cpa(void* s, const void* g) { asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(su(s)), "l"(g)); }
DEV void commit() { asm volatile("cp.async.commit_group;\n" ::); }
DEV void wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }
constexpr int GB = 64, GK = 16, LMK = 68, LKM = 20, TD = 1280;
template <bool LOADC, bool STOREC, bool SMEMEPI>
__global__ void __launch_bounds__(128) k(const double* A, const double* B, double* C, int M, int N, int K) {
  extern __shared__ __align__(16) double sm[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gq = lane >> 2, tq = lane & 3;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32, m0 = blockIdx.x * GB, n0 = blockIdx.y * GB;
  const long z = blockIdx.z;
  const long sA = (long)M * K, sB = (long)K * N, sC = (long)M * N;
  const double* Ar = A + z * 2 * sA; const double* Ai = Ar + sA;
  const double* Br = B + z * 2 * sB; const double* Bi = Br + sB;
  double* Cr = C + z * 2 * sC; double* Ci = Cr + sC;
  auto issue = [&](int st, int kt) {
    double* b = sm + st * 4 * TD;
    for (int i = 0; i < 4; ++i) { int c = tid + i * 128, col = c >> 5, ch = c & 31;
      cpa(b + col * LMK + ch * 2, Ar + (long)(kt * GK + col) * M + m0 + ch * 2);
      cpa(b + TD + col * LMK + ch * 2, Ai + (long)(kt * GK + col) * M + m0 + ch * 2); }
    for (int i = 0; i < 4; ++i) { int c = tid + i * 128, col = c >> 3, ch = c & 7;
      cpa(b + 2 * TD + col * LKM + ch * 2, Br + (long)(n0 + col) * K + kt * GK + ch * 2);
      cpa(b + 3 * TD + col * LKM + ch * 2, Bi + (long)(n0 + col) * K + kt * GK + ch * 2); }
  };
  const int KT = K / GK;
  issue(0, 0); commit();
  double ar_[4][4][2], ai_[4][4][2];
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) for (int e = 0; e < 2; ++e) {
    long off = (long)(n0 + wn + j * 8 + 2 * tq + e) * M + m0 + wm + i * 8 + gq;
    ar_[i][j][e] = LOADC ? Cr[off] : 0.0; ai_[i][j][e] = LOADC ? Ci[off] : 0.0; }
  for (int kt = 0; kt < KT; ++kt) {
    wait0(); __syncthreads();
    if (kt + 1 < KT) issue((kt + 1) & 1, kt + 1);
    commit();
    const double* b = sm + (kt & 1) * 4 * TD;
    for (int kk = 0; kk < GK; kk += 4) {
      double a[4], c[4], nc[4], br[4], bi[4];
      for (int i = 0; i < 4; ++i) { a[i] = -b[(kk + tq) * LMK + wm + i * 8 + gq]; c[i] = -b[TD + (kk + tq) * LMK + wm + i * 8 + gq]; nc[i] = -c[i]; }
      for (int j = 0; j < 4; ++j) { br[j] = b[2 * TD + (wn + j * 8 + gq) * LKM + kk + tq]; bi[j] = b[3 * TD + (wn + j * 8 + gq) * LKM + kk + tq]; }
      for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) dmma(ar_[i][j], a[i], br[j]);
      for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) dmma(ai_[i][j], a[i], bi[j]);
      for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) dmma(ar_[i][j], nc[i], bi[j]);
      for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) dmma(ai_[i][j], c[i], br[j]);
    }
    __syncthreads();
  }
  if (!STOREC) { if (ar_[0][0][0] == 1.2345) Cr[0] = 1; return; }
  if (!SMEMEPI) {
    for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) for (int e = 0; e < 2; ++e) {
      long off = (long)(n0 + wn + j * 8 + 2 * tq + e) * M + m0 + wm + i * 8 + gq;
      Cr[off] = ar_[i][j][e]; Ci[off] = ai_[i][j][e]; }
  } else {
    double* cr = sm; double* ci = sm + 64 * 66;
    for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) for (int e = 0; e < 2; ++e) {
      int o = (wn + j * 8 + 2 * tq + e) * 66 + wm + i * 8 + gq; cr[o] = ar_[i][j][e]; ci[o] = ai_[i][j][e]; }
    __syncthreads();
    for (int c = tid; c < 64 * 32; c += 128) { int col = c >> 5, ch = c & 31;
      double2 v = *(double2*)(cr + col * 66 + ch * 2); *(double2*)(Cr + (long)(n0 + col) * M + m0 + ch * 2) = v;
      double2 w = *(double2*)(ci + col * 66 + ch * 2); *(double2*)(Ci + (long)(n0 + col) * M + m0 + ch * 2) = w; }
  }
}
template <bool L, bool S, bool E> void run(const char* name, double* A, double* B, double* C, int M, int N, int K, int bt) {
  size_t sm = 2 * 4 * TD * 8;
  cudaFuncSetAttribute(k<L, S, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  dim3 g(M / 64, N / 64, bt);
  k<L, S, E><<<g, 128, sm>>>(A, B, C, M, N, K);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); for (int i = 0; i < 10; ++i) k<L, S, E><<<g, 128, sm>>>(A, B, C, M, N, K); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
  double fl = 8.0 * M * N * K * bt;
  printf("%-28s K=%4d: %.3f ms %.2f TF/s (%.1f%%) %s\n", name, K, ms, fl / ms / 1e9, 100 * fl / ms / 1e9 / 37.08, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  int M = 4032, N = 4032, bt = 4;
  for (int K : {64, 128, 1024}) {
    double *A, *B, *C;
    cudaMalloc(&A, 2l * M * K * bt * 8); cudaMalloc(&B, 2l * K * N * bt * 8); cudaMalloc(&C, 2l * M * N * bt * 8);
    cudaMemset(A, 0, 2l * M * K * bt * 8); cudaMemset(B, 0, 2l * K * N * bt * 8); cudaMemset(C, 0, 2l * M * N * bt * 8);
    run<true, true, false>("load C, store C (current)", A, B, C, M, N, K, bt);
    run<false, true, false>("no C load", A, B, C, M, N, K, bt);
    run<true, false, false>("no C store", A, B, C, M, N, K, bt);
    run<false, false, false>("no C load, no store", A, B, C, M, N, K, bt);
    run<true, true, true>("load C, smem-staged store", A, B, C, M, N, K, bt);
    cudaFree(A); cudaFree(B); cudaFree(C);
  }
}
