// reduce.cu — generic Collect (map / zipWith) and Reduce / MapReduce families over dense
// vectors: axpy (collect), sum (fp64 / int64), the fused mean_variance loop (two reduce
// elems sharing one traversal) and count_where (predicated reduce).
//
// Reference lowering: emit_parallel_loop (proj/src/codegen.cpp:345-433): collect stores
// out(i) = v, reduce folds acc = combine(acc, v) under its cond guard.  Device plan:
// grid-stride with 128-bit loads, per-thread fold, warp shuffle tree, per-CTA partial,
// ascending-CTA final combine (deterministic for a given device).
#include <algorithm>

#include "common.cuh"

namespace dlx {

constexpr int kRedThreads = 256;

static int red_grid(int64_t n) {
  int64_t grid = static_cast<int64_t>(sm_count()) * 4;
  const int64_t need = (n + 2 * kRedThreads - 1) / (2 * kRedThreads);
  return static_cast<int>(std::max<int64_t>(1, std::min(grid, need)));
}

__global__ void axpy_kernel(double a, const double* __restrict__ x, const double* __restrict__ y,
                            int64_t n, double* __restrict__ out) {
  // MiniC `a * x(i) + y(i)`: two roundings, no FMA (SPEC.md:642 demands exact equality)
  const int64_t T = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += T)
    out[i] = __dadd_rn(__dmul_rn(a, x[i]), y[i]);
}

__global__ void widen_kernel(const int32_t* __restrict__ a, int64_t n, long long* __restrict__ out) {
  const int64_t T = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += T)
    out[i] = a[i];
}

__global__ void axpy_inplace_kernel(double* __restrict__ t, const double* __restrict__ g,
                                    double alpha, int64_t n) {
  pdl_wait();   // programmatic dependent launch: inputs are final from here on
  pdl_trigger();
  const int64_t T = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += T)
    t[i] = __dsub_rn(t[i], __dmul_rn(alpha, g[i]));
}

enum RedOp { kSumF64 = 0, kSumSqF64 = 1, kCountGt = 2, kSumI64 = 3 };

// Partial per CTA: out[blockIdx*W + w], W = 2 for sum/sumsq, 1 otherwise.
template <int OP>
__global__ void __launch_bounds__(kRedThreads)
reduce_kernel(const void* __restrict__ src, int64_t n, double thr, void* __restrict__ parts) {
  __shared__ double sd[2][kRedThreads / 32];
  __shared__ long long sl[kRedThreads / 32];
  const int64_t T = static_cast<int64_t>(gridDim.x) * kRedThreads;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * kRedThreads + threadIdx.x;
  double a = 0.0, b = 0.0;
  long long c = 0;
  if (OP == kSumI64) {
    const long long* x = static_cast<const long long*>(src);
    for (int64_t i = tid; i < n; i += T) c += __ldg(x + i);
  } else {
    const double* x = static_cast<const double*>(src);
    const int64_t np = n >> 1;
    const double2* x2 = reinterpret_cast<const double2*>(x);
    for (int64_t q = tid; q < np; q += T) {
      const double2 v = __ldg(x2 + q);
      if (OP == kCountGt) {
        c += (thr < v.x) + (thr < v.y);
      } else {
        a += v.x;
        a += v.y;
        if (OP == kSumSqF64) {
          b += v.x * v.x;
          b += v.y * v.y;
        }
      }
    }
    if ((n & 1) && tid == 0) {
      const double v = x[n - 1];
      if (OP == kCountGt) c += (thr < v);
      else { a += v; if (OP == kSumSqF64) b += v * v; }
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  c = warp_sum_ll(c);
  if (lane == 0) { sd[0][warp] = a; sd[1][warp] = b; sl[warp] = c; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double ta = sd[0][0], tb = sd[1][0];
    long long tc = sl[0];
    for (int w = 1; w < kRedThreads / 32; ++w) { ta += sd[0][w]; tb += sd[1][w]; tc += sl[w]; }
    if (OP == kSumF64) static_cast<double*>(parts)[blockIdx.x] = ta;
    if (OP == kSumSqF64) {
      static_cast<double*>(parts)[2 * blockIdx.x] = ta;
      static_cast<double*>(parts)[2 * blockIdx.x + 1] = tb;
    }
    if (OP == kCountGt || OP == kSumI64) static_cast<long long*>(parts)[blockIdx.x] = tc;
  }
}

template <int OP>
__global__ void reduce_final_kernel(const void* __restrict__ parts, int nparts, void* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (OP == kSumF64) {
    const double* p = static_cast<const double*>(parts);
    double a = p[0];
    for (int i = 1; i < nparts; ++i) a += p[i];
    *static_cast<double*>(out) = a;
  } else if (OP == kSumSqF64) {
    const double* p = static_cast<const double*>(parts);
    double a = p[0], b = p[1];
    for (int i = 1; i < nparts; ++i) { a += p[2 * i]; b += p[2 * i + 1]; }
    static_cast<double*>(out)[0] = a;
    static_cast<double*>(out)[1] = b;
  } else {
    const long long* p = static_cast<const long long*>(parts);
    long long a = 0;
    for (int i = 0; i < nparts; ++i) a += p[i];
    *static_cast<long long*>(out) = a;
  }
}

template <int OP>
static int run_reduce(const void* src, int64_t n, double thr, void* out, void* ws, size_t wsb,
                      cudaStream_t stream) {
  DLX_REQUIRE(n >= 0 && out && (src || n == 0), DLX_ERR_ARG, "reduce: bad args");
  DLX_REQUIRE((reinterpret_cast<uintptr_t>(src) & 15) == 0, DLX_ERR_ARG,
              "reduce: input must be 16-byte aligned");
  const int grid = red_grid(n);
  DLX_REQUIRE(ws && wsb >= static_cast<size_t>(grid) * 16, DLX_ERR_ARG, "reduce: workspace too small");
  reduce_kernel<OP><<<grid, kRedThreads, 0, stream>>>(src, n, thr, ws);
  DLX_LAUNCHED("reduce_kernel");
  reduce_final_kernel<OP><<<1, 32, 0, stream>>>(ws, grid, out);
  DLX_LAUNCHED("reduce_final_kernel");
  return DLX_OK;
}

}  // namespace dlx

using namespace dlx;

extern "C" {

int dlx_map_axpy(double a, const double* d_x, const double* d_y, int64_t n, double* d_out,
                 dlx_stream_t stream) {
  DLX_REQUIRE(n >= 0 && ((d_x && d_y && d_out) || n == 0), DLX_ERR_ARG, "axpy: bad args");
  if (n == 0) return DLX_OK;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, sm_count() * 8));
  axpy_kernel<<<grid, 256, 0, stream>>>(a, d_x, d_y, n, d_out);
  DLX_LAUNCHED("axpy_kernel");
  return DLX_OK;
}

int dlx_axpy_inplace(double* d_theta, const double* d_grad, double alpha, int64_t n,
                     dlx_stream_t stream) {
  DLX_REQUIRE(n >= 0 && ((d_theta && d_grad) || n == 0), DLX_ERR_ARG, "axpy_inplace: bad args");
  if (n == 0) return DLX_OK;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, sm_count() * 8));
  DLX_CUDA(launch_pdl(axpy_inplace_kernel, dim3(grid), dim3(256), 0, stream, d_theta, d_grad, alpha, n));
  DLX_LAUNCHED("axpy_inplace_kernel");
  return DLX_OK;
}

int dlx_widen_i32_i64(const int32_t* d_in, int64_t n, int64_t* d_out, dlx_stream_t stream) {
  DLX_REQUIRE(n >= 0 && ((d_in && d_out) || n == 0), DLX_ERR_ARG, "widen: bad args");
  if (n == 0) return DLX_OK;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, sm_count() * 8));
  widen_kernel<<<grid, 256, 0, stream>>>(d_in, n, reinterpret_cast<long long*>(d_out));
  DLX_LAUNCHED("widen_kernel");
  return DLX_OK;
}

size_t dlx_reduce_workspace_bytes(int64_t n) { return static_cast<size_t>(red_grid(n)) * 16 + 256; }

int dlx_reduce_sum_f64(const double* d_x, int64_t n, double* d_out, void* ws, size_t wsb,
                       dlx_stream_t stream) {
  return run_reduce<kSumF64>(d_x, n, 0.0, d_out, ws, wsb, stream);
}
int dlx_reduce_sum_i64(const int64_t* d_x, int64_t n, int64_t* d_out, void* ws, size_t wsb,
                       dlx_stream_t stream) {
  return run_reduce<kSumI64>(d_x, n, 0.0, d_out, ws, wsb, stream);
}
int dlx_reduce_sum_sumsq_f64(const double* d_x, int64_t n, double* d_out2, void* ws, size_t wsb,
                             dlx_stream_t stream) {
  return run_reduce<kSumSqF64>(d_x, n, 0.0, d_out2, ws, wsb, stream);
}
int dlx_reduce_count_gt_f64(const double* d_x, int64_t n, double thr, int64_t* d_out, void* ws,
                            size_t wsb, dlx_stream_t stream) {
  return run_reduce<kCountGt>(d_x, n, thr, d_out, ws, wsb, stream);
}

}  // extern "C"
