// microbenchmark: throughput of fp64 -> int64 conversion vs the magic-number DFMA split
#include <cstdio>
#include <cstdint>
__global__ void conv_f2i(const double* __restrict__ x, unsigned long long* out, int iters) {
  double v = x[threadIdx.x] , s = 1099511627776.0;
  unsigned long long acc = 0;
  double a0 = v, a1 = v * 1.1, a2 = v * 1.3, a3 = v * 1.7;
  for (int i = 0; i < iters; ++i) {
    acc += (unsigned long long)__double2ll_rd(a0 * s) + (unsigned long long)__double2ll_rd(a1 * s) +
           (unsigned long long)__double2ll_rd(a2 * s) + (unsigned long long)__double2ll_rd(a3 * s);
    a0 += 1e-9; a1 += 1e-9; a2 += 1e-9; a3 += 1e-9;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void conv_magic(const double* __restrict__ x, unsigned long long* out, int iters) {
  double v = x[threadIdx.x], s = 256.0;
  const double M = 6755399441055744.0;
  unsigned long long acc = 0;
  double a0 = v, a1 = v * 1.1, a2 = v * 1.3, a3 = v * 1.7;
  for (int i = 0; i < iters; ++i) {
    double t[4] = {a0, a1, a2, a3};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      double t1 = __fma_rd(t[e], s, M), hd = t1 - M, r = __fma_rn(t[e], s, -hd), t2 = __fma_rd(r, 4294967296.0, M);
      acc += (unsigned)__double2loint(t1) + (unsigned)__double2loint(t2);
    }
    a0 += 1e-9; a1 += 1e-9; a2 += 1e-9; a3 += 1e-9;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  double* x; unsigned long long* o;
  cudaMalloc(&x, 8 * 1024); cudaMalloc(&o, 8 * 148 * 4 * 512);
  cudaMemset(x, 0, 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096, blocks = 148 * 4, threads = 512;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0); conv_f2i<<<blocks, threads>>>(x, o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double n = 4.0 * iters * blocks * threads;
    printf("f2i.s64 (dmul+f2i): %.3f ms, %.2f G conv/s, %.2f conv/clk/SM @1.965GHz\n", ms, n / ms / 1e6, n / (ms * 1e-3) / 148 / 1.965e9);
    cudaEventRecord(e0); conv_magic<<<blocks, threads>>>(x, o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("magic 4-DP split: %.3f ms, %.2f G conv/s, %.2f conv/clk/SM\n", ms, n / ms / 1e6, n / (ms * 1e-3) / 148 / 1.965e9);
  }
  return 0;
}
