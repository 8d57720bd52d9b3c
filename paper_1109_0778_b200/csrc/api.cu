// api.cu — error state, device/memory/stream plumbing and the synthetic Rng sources.
#include <atomic>
#include <cstdarg>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace dlx {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

int sm_count() {
  static std::mutex mu;
  static std::vector<int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  std::lock_guard<std::mutex> lock(mu);
  if (dev >= static_cast<int>(cache.size())) cache.resize(dev + 1, 0);
  if (cache[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    cache[dev] = v;
  }
  return cache[dev];
}

// ---------------------------------------------------------------------------------------
// Rng sources (runtime.hpp:86-96).  Thread t of the grid owns elements t, t+T, t+2T, ...
// (T = total threads) so stores are coalesced; its first state comes from an O(log n)
// skip-ahead and each later element is one affine step of stride T.

template <bool kInt>
__global__ void rng_kernel(void* out, int64_t n, int64_t bound, uint64_t seed,
                           uint64_t first_draw, uint64_t stride_mul, uint64_t stride_add) {
  const int64_t T = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n) return;
  // state *after* draw number (first_draw + e): advance seed by first_draw + e + 1 steps
  uint64_t s = rng_advance(seed, first_draw + static_cast<uint64_t>(e) + 1);
  const double b = static_cast<double>(bound);
  for (; e < n; e += T) {
    const double u = static_cast<double>(s >> 11) * 0x1.0p-53;
    if (kInt)
      static_cast<int64_t*>(out)[e] = static_cast<int64_t>(u * b);
    else
      static_cast<double*>(out)[e] = u;
    s = stride_mul * s + stride_add;
  }
}

template <bool kInt>
static int launch_rng(void* out, int64_t n, int64_t bound, uint64_t seed, uint64_t first_draw,
                      dlx_stream_t stream) {
  DLX_REQUIRE(n >= 0, DLX_ERR_ARG, "rng: negative length %lld", (long long)n);
  DLX_REQUIRE(out != nullptr || n == 0, DLX_ERR_ARG, "rng: null output");
  if (n == 0) return DLX_OK;
  const int threads = 256;
  int64_t blocks = static_cast<int64_t>(sm_count()) * 8;
  const int64_t need = (n + threads - 1) / threads;
  if (blocks > need) blocks = need;
  const uint64_t T = static_cast<uint64_t>(blocks) * threads;
  // affine map for T steps: s -> A*s + C  (rng_advance(s, T) = A*s + C)
  const uint64_t C = rng_advance(0, T);
  const uint64_t A = rng_advance(1, T) - C;
  rng_kernel<kInt><<<static_cast<unsigned>(blocks), threads, 0, stream>>>(out, n, bound, seed,
                                                                            first_draw, A, C);
  DLX_LAUNCHED("rng_kernel");
  return DLX_OK;
}

static std::atomic<unsigned long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

}  // namespace dlx

using namespace dlx;

extern "C" {

const char* dlx_last_error(void) { return g_last_error.c_str(); }
uint64_t dlx_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }
const char* dlx_version(void) { return "dlx 0.1 (sm_100a)"; }

int dlx_device_count(int* count) {
  DLX_REQUIRE(count, DLX_ERR_ARG, "null count");
  DLX_CUDA(cudaGetDeviceCount(count));
  return DLX_OK;
}
int dlx_set_device(int device) {
  DLX_CUDA(cudaSetDevice(device));
  return DLX_OK;
}
int dlx_sm_count(int* sms) {
  DLX_REQUIRE(sms, DLX_ERR_ARG, "null sms");
  *sms = sm_count();
  return DLX_OK;
}
int dlx_malloc(void** d_ptr, size_t bytes) {
  DLX_REQUIRE(d_ptr, DLX_ERR_ARG, "null d_ptr");
  DLX_CUDA(cudaMalloc(d_ptr, bytes ? bytes : 1));
  return DLX_OK;
}
int dlx_free(void* d_ptr) {
  DLX_CUDA(cudaFree(d_ptr));
  return DLX_OK;
}
int dlx_host_alloc(void** h_ptr, size_t bytes) {
  DLX_REQUIRE(h_ptr, DLX_ERR_ARG, "null h_ptr");
  DLX_CUDA(cudaMallocHost(h_ptr, bytes ? bytes : 1));
  return DLX_OK;
}
int dlx_host_free(void* h_ptr) {
  DLX_CUDA(cudaFreeHost(h_ptr));
  return DLX_OK;
}
int dlx_memcpy_h2d(void* d_dst, const void* h_src, size_t bytes, dlx_stream_t stream) {
  DLX_CUDA(cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice, stream));
  return DLX_OK;
}
int dlx_memcpy_d2h(void* h_dst, const void* d_src, size_t bytes, dlx_stream_t stream) {
  DLX_CUDA(cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost, stream));
  return DLX_OK;
}
int dlx_memset(void* d_dst, int value, size_t bytes, dlx_stream_t stream) {
  DLX_CUDA(cudaMemsetAsync(d_dst, value, bytes, stream));
  return DLX_OK;
}
int dlx_stream_create(dlx_stream_t* stream) {
  DLX_REQUIRE(stream, DLX_ERR_ARG, "null stream");
  cudaStream_t s;
  DLX_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  *stream = s;
  return DLX_OK;
}
int dlx_stream_destroy(dlx_stream_t stream) {
  DLX_CUDA(cudaStreamDestroy(stream));
  return DLX_OK;
}
int dlx_stream_sync(dlx_stream_t stream) {
  DLX_CUDA(cudaStreamSynchronize(stream));
  return DLX_OK;
}

int dlx_rng_units(double* d_out, int64_t n, uint64_t seed, uint64_t first_draw,
                  dlx_stream_t stream) {
  return launch_rng<false>(d_out, n, 0, seed, first_draw, stream);
}
int dlx_rng_ints(int64_t* d_out, int64_t n, int64_t bound, uint64_t seed, uint64_t first_draw,
                 dlx_stream_t stream) {
  return launch_rng<true>(d_out, n, bound, seed, first_draw, stream);
}

}  // extern "C"
