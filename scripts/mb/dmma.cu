// DMMA (fp64 tensor core) throughput microbenchmark: independent accumulator chains per warp,
// no memory traffic.  Reports TFLOP/s for mma.sync f64 shapes m8n8k4, m16n8k4, m16n8k8, m16n8k16.
#include <cstdio>
#include <cuda_runtime.h>

template <int kShape, int kChains>
__global__ void dmma_loop(double* out, int iters) {
  double a[8], b[4], c[kChains][4];
  for (int i = 0; i < 8; ++i) a[i] = 1e-3 * (threadIdx.x + i);
  for (int i = 0; i < 4; ++i) b[i] = 1e-3 * (threadIdx.x - i);
  for (int q = 0; q < kChains; ++q) for (int i = 0; i < 4; ++i) c[q][i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < kChains; ++q) {
      if (kShape == 0)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a[0]), "d"(b[0]));
      else if (kShape == 1)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[q][0]), "+d"(c[q][1]), "+d"(c[q][2]), "+d"(c[q][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      else if (kShape == 2)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(c[q][0]), "+d"(c[q][1]), "+d"(c[q][2]), "+d"(c[q][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(c[q][0]), "+d"(c[q][1]), "+d"(c[q][2]), "+d"(c[q][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
  for (int q = 0; q < kChains; ++q) for (int i = 0; i < 4; ++i) s += c[q][i];
  if (s == 12345.0) out[0] = s;
}

template <int kShape, int kChains>
void run(const char* name, double flop_per_mma, int warps_per_block) {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  dim3 grid(sms), block(32 * warps_per_block);
  dmma_loop<kShape, kChains><<<grid, block>>>(out, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  dmma_loop<kShape, kChains><<<grid, block>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = flop_per_mma * kChains * iters * (double)warps_per_block * sms;
  printf("%-10s chains=%d warps/SM=%2d : %.2f TFLOP/s (%.3f ms) %s\n", name, kChains, warps_per_block,
         flops / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0, 4>("m8n8k4", 2.0 * 8 * 8 * 4, w);
    run<0, 8>("m8n8k4", 2.0 * 8 * 8 * 4, w);
    run<1, 4>("m16n8k4", 2.0 * 16 * 8 * 4, w);
    run<2, 4>("m16n8k8", 2.0 * 16 * 8 * 8, w);
    run<3, 4>("m16n8k16", 2.0 * 16 * 8 * 16, w);
  }
  return 0;
}
