// common.cuh — shared helpers for the dlx CUDA sources (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/dlx.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "dlx kernels target sm_100a only"
#endif

namespace dlx {

// Thread-local last-error text, returned by dlx_last_error().
void set_error(const char* fmt, ...);

// Kernels launched by this library since load (incremented by DLX_LAUNCHED on success):
// the bench reports it as gpu_launches, evidence that the native path ran.
void count_launch();

inline int cuda_fail(cudaError_t e, const char* what) {
  set_error("%s: %s", what, cudaGetErrorString(e));
  return DLX_ERR_CUDA;
}

#define DLX_CUDA(call)                                    \
  do {                                                    \
    cudaError_t _e = (call);                              \
    if (_e != cudaSuccess) return ::dlx::cuda_fail(_e, #call); \
  } while (0)

#define DLX_LAUNCHED(name)                                \
  do {                                                    \
    cudaError_t _e = cudaGetLastError();                  \
    if (_e != cudaSuccess) return ::dlx::cuda_fail(_e, name); \
    ::dlx::count_launch();                                \
  } while (0)

#define DLX_REQUIRE(cond, code, ...)                      \
  do {                                                    \
    if (!(cond)) {                                        \
      ::dlx::set_error(__VA_ARGS__);                      \
      return (code);                                      \
    }                                                     \
  } while (0)

// Deterministic combine of per-CTA partial activation records (combine.cu).
int combine_f64(const double* parts, int nparts, long long width, double* out, cudaStream_t s);
int combine_i64(const long long* parts, int nparts, long long width, long long* out, cudaStream_t s);
// an fp64 and an int64 record (same number of partials) in one launch
int combine_kmeans_update(const double* pf, double* of, const long long* pi, long long* oi, int k, int d,
                          int nparts, double* mu, cudaStream_t s);
int combine_f64_i64(const double* pf, long long wf, double* of, const long long* pi, long long wi,
                    long long* oi, int nparts, cudaStream_t s);
int combine_u32_i64(const unsigned* parts, int nparts, long long width, long long* out, cudaStream_t s);
// combine_f64 that does nothing when the device flag *d_skip is set when it runs
int combine_f64_unless(const double* parts, int nparts, long long width, double* out,
                       const int* d_skip, cudaStream_t s);

// Programmatic dependent launch (PDL): a kernel launched with launch_pdl may start while the
// previous kernel on the stream is still running; it must call pdl_wait() before touching
// anything that kernel writes (or that the kernel before it reads).  Both are no-ops for a
// normal launch.  pdl_trigger() lets the next PDL kernel start early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Number of SMs of the current device (cached per device).
int sm_count();

// Workspace carving: 256-byte aligned sub-allocations out of one caller buffer.
struct Carve {
  char* base;
  size_t used = 0;
  __host__ __device__ explicit Carve(void* p) : base(static_cast<char*>(p)) {}
  template <class T>
  __host__ __device__ T* take(size_t count) {
    used = (used + 255) & ~size_t(255);
    T* p = reinterpret_cast<T*>(base ? base + used : nullptr);
    used += count * sizeof(T);
    return p;
  }
};

// LCG constants of the reference Rng (runtime.hpp:90).
constexpr uint64_t kRngMul = 6364136223846793005ULL;
constexpr uint64_t kRngInc = 1442695040888963407ULL;

__host__ __device__ inline uint64_t rng_advance(uint64_t state, uint64_t n) {
  uint64_t am = 1, aa = 0, cm = kRngMul, ca = kRngInc;
  while (n) {
    if (n & 1) {
      am = am * cm;
      aa = aa * cm + ca;
    }
    ca = (cm + 1) * ca;
    cm = cm * cm;
    n >>= 1;
  }
  return am * state + aa;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Streaming 128-bit load that does not allocate in L1 (each sample row is read once).
__device__ __forceinline__ double2 ld_stream_f64x2(const double* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p));
  return r;
}

}  // namespace dlx
