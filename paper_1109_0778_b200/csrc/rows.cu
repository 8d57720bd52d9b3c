// rows.cu — row-streaming multiloops over a row-major DenseMatrix: the logistic-regression
// gradient and GDA passes 1 and 2 (§8 a6).
//
// Shared device plan for the streaming families: a warp streams blocks of 8 consecutive
// rows, lane l holding columns {2l, 2l+1} + 64m of each (128-bit loads, so a d=64 fp64 row is
// one warp-wide load and 8 are in flight per lane); every reduce slot that all samples feed (gradient,
// per-class sums) is a per-lane register accumulator, reduced across warps through shared
// memory in ascending warp order, written as a per-CTA partial and folded across CTAs by the
// deterministic combine kernel (combine.cu).  Pass 2 (d <= 64) runs on the fp64 tensor cores
// (gda_dmma.cu); the CUDA-core register-tile kernel below covers 64 < d <= 128.
#include <algorithm>

#include <cstdlib>
#include <utility>

#include "common.cuh"

namespace dlx {

constexpr int kRowThreads = 256;
constexpr int kRowWarps = kRowThreads / 32;
constexpr int kMaxM = 4;  // 128-bit column groups per lane => d <= 64*kMaxM

// One full wave of 2 CTAs per SM (16 warps, up to 128 registers per thread).  The earlier
// 4 CTAs per SM grid against a 3-CTA register occupancy left a quarter of the work to a
// second, 1-CTA wave: logreg L16 92 % -> 107 % of the copy peak, C2 65 % -> 98 % (profiles r77-r78).
#ifndef DLX_ROW_GRID_MULT
#define DLX_ROW_GRID_MULT 2
#endif
#ifndef DLX_ROW_MINB
#define DLX_ROW_MINB 2
#endif
static int row_grid(int64_t n) {
  int64_t grid = static_cast<int64_t>(sm_count()) * DLX_ROW_GRID_MULT;
  const int64_t need = (n + kRowWarps - 1) / kRowWarps;
  return static_cast<int>(std::max<int64_t>(1, std::min(grid, need)));
}

// CTA-wide ascending-warp reduction of per-lane column accumulators into out[d].
template <int M>
__device__ void cta_reduce_columns(double (&acc)[M][2], int d, double* red_s, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int j = 64 * m + 2 * lane;
    if (j < d) red_s[warp * d + j] = acc[m][0];
    if (j + 1 < d) red_s[warp * d + j + 1] = acc[m][1];
  }
  __syncthreads();
  for (int j = threadIdx.x; j < d; j += kRowThreads) {
    double v = red_s[j];
    for (int w = 1; w < kRowWarps; ++w) v += red_s[w * d + j];
    out[j] = v;
  }
  __syncthreads();
}

// 8 rows in flight per warp: lane l holds columns {2l, 2l+1} + 64m of rows r0..r0+7.
constexpr int kRows = 8;
#ifndef DLX_F32_GROUPS
#define DLX_F32_GROUPS 2   // fp32 storage, d <= 64: blocks of 8 rows in flight per warp step
#endif

// fp32 storage (the opt-in mode): two floats per lane, kept packed in registers
// (so a warp keeps twice the rows in flight for the same registers) and promoted exactly to fp64
// at use
__device__ __forceinline__ float2 ld_stream_f32x2(const float* p) {
  float2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
  return r;
}
template <int M>
__device__ __forceinline__ void load_rows(const float* __restrict__ x, int64_t i0, int64_t n, int d,
                                          int lane, float2 (&v)[kRows][M]) {
#pragma unroll
  for (int r = 0; r < kRows; ++r) {
    const int64_t i = i0 + r;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int j = 64 * m + 2 * lane;
      v[r][m] = (i < n && j < d) ? ld_stream_f32x2(x + i * d + j) : make_float2(0.f, 0.f);
    }
  }
}
__device__ __forceinline__ double2 to_d2(double2 v) { return v; }
// float -> double, exact: for normal floats the double's words are built with integer ops
// (exponent rebias +896, mantissa << 29) instead of F2F.F64.F32, whose throughput bounded the
// fp32 kernel; zero, subnormal, inf and NaN take the conversion instruction
__device__ __forceinline__ double f2d_exact(float f) {
  const uint32_t u = __float_as_uint(f), em = u & 0x7fffffffu;
  if (em - 0x00800000u < 0x7f000000u)   // 0 < exponent < 255
    return __hiloint2double(static_cast<int>((u & 0x80000000u) | ((em >> 3) + 0x38000000u)), static_cast<int>(em << 29));
  return static_cast<double>(f);
}
__device__ __forceinline__ double2 to_d2(float2 v) { return make_double2(f2d_exact(v.x), f2d_exact(v.y)); }
template <class T> struct Vec2;
template <> struct Vec2<double> { using type = double2; };
template <> struct Vec2<float> { using type = float2; };

template <int M>
__device__ __forceinline__ void load_rows(const double* __restrict__ x, int64_t i0, int64_t n, int d,
                                          int lane, double2 (&v)[kRows][M]) {
#pragma unroll
  for (int r = 0; r < kRows; ++r) {
    const int64_t i = i0 + r;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int j = 64 * m + 2 * lane;
      v[r][m] = (i < n && j < d) ? ld_stream_f64x2(x + i * d + j) : make_double2(0.0, 0.0);
    }
  }
}

// Reduce-scatter of 8 per-lane partial dot products: 9 fp64 shuffles instead of 8 x 5.
// Returns the full dot of row  row_of_lane(lane) = 4*b4 + 2*b3 + b2  (b_k = bit k of lane);
// every row ends up on the 4 lanes that differ in bits 0-1.
__device__ __forceinline__ double reduce_scatter8(const double (&p)[kRows], int lane) {
  const bool b4 = (lane >> 4) & 1, b3 = (lane >> 3) & 1, b2 = (lane >> 2) & 1;
  double q4[4], q2[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double send = b4 ? p[i] : p[i + 4];
    const double keep = b4 ? p[i + 4] : p[i];
    q4[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const double send = b3 ? q4[i] : q4[i + 2];
    const double keep = b3 ? q4[i + 2] : q4[i];
    q2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  const double send = b2 ? q2[0] : q2[1];
  const double keep = b2 ? q2[1] : q2[0];
  double z = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  z += __shfl_xor_sync(0xffffffffu, z, 2);
  z += __shfl_xor_sync(0xffffffffu, z, 1);
  return z;
}

__device__ __forceinline__ int lane_of_row(int r) {
  return (((r >> 2) & 1) << 4) | (((r >> 1) & 1) << 3) | ((r & 1) << 2);
}

// ---------------------------------------------------------------------------------------
// logistic regression: g_j = sum_i (link(theta . x_i) - y_i) x_ij
// One fused pass: dot (FMA partials + reduce-scatter), the link once per row on 4 lanes
// (optionally stored: the staged program's collect h(i) = link(theta . x_i)), residual
// broadcast, gradient FMAs into per-lane registers.  Link = the sigmoid of the family API, or a
// link expression compiled by the executor from the loop body (LinkCode: the reference has no
// exp, so staged programs carry their own link, e.g. softsign t / (1 + |t|)).
struct SigmoidLink {
  __device__ __forceinline__ double operator()(double z) const { return 1.0 / (1.0 + exp(-z)); }
};
struct SoftsignLink {
  __device__ __forceinline__ double operator()(double z) const { return z / (1.0 + fabs(z)); }
};
// The link code as an expression over t (r[0]): the canonical sigmoid 1 / (1 + exp(0 - t)) and
// softsign t / (1 + |t|) that staged logistic-regression loops carry run as the fixed functors
// above (the same IEEE operations in the same order, so bit-identical: 0 - t and -t differ only
// in the sign of a zero, and exp(+0) = exp(-0)); any other code runs the interpreted CodeLink.
enum LinkKind { kLinkCode = 0, kLinkSigmoid = 1, kLinkSoftsign = 2 };
static bool link_const(const dlx_link_code& c, int q, double v) { return c.op[q] == DLX_LINK_CONST && c.imm[q] == v; }
// the instruction that last wrote register r before instruction q (-1: the input t when r == 0)
static int link_def(const dlx_link_code& c, int r, int q) {
  for (int p = q - 1; p >= 0; --p)
    if (c.dst[p] == r) return p;
  return r == 0 ? -1 : -2;
}
static LinkKind link_kind(const dlx_link_code& c) {
  const int top = link_def(c, c.out, c.n);
  if (top < 0 || c.op[top] != DLX_LINK_DIV) return kLinkCode;
  const int num = link_def(c, c.a[top], top), den = link_def(c, c.b[top], top);
  if (den < 0 || c.op[den] != DLX_LINK_ADD) return kLinkCode;
  int l = link_def(c, c.a[den], den), r = link_def(c, c.b[den], den);
  if (l >= 0 && !link_const(c, l, 1.0)) std::swap(l, r);
  if (l < 0 || !link_const(c, l, 1.0) || r < 0) return kLinkCode;
  if (num >= 0 && link_const(c, num, 1.0) && c.op[r] == DLX_LINK_EXP) {       // 1 / (1 + exp(0 - t))
    const int sub = link_def(c, c.a[r], r);
    if (sub < 0 || c.op[sub] != DLX_LINK_SUB) return kLinkCode;
    const int z = link_def(c, c.a[sub], sub), t = link_def(c, c.b[sub], sub);
    return (z >= 0 && link_const(c, z, 0.0) && t == -1) ? kLinkSigmoid : kLinkCode;
  }
  if (num == -1 && c.op[r] == DLX_LINK_ABS && link_def(c, c.a[r], r) == -1) return kLinkSoftsign;   // t / (1 + |t|)
  return kLinkCode;
}

struct CodeLink {
  dlx_link_code c;
  // registers: r[0] = t; every instruction writes r[dst]; IEEE round-to-nearest, no contraction
  __device__ double operator()(double t) const {
    double r[DLX_LINK_MAX_REGS];
    r[0] = t;
    for (int q = 0; q < c.n; ++q) {
      const double a = r[c.a[q]], b = r[c.b[q]];
      double v;
      switch (c.op[q]) {
        case DLX_LINK_CONST: v = c.imm[q]; break;
        case DLX_LINK_ADD: v = __dadd_rn(a, b); break;
        case DLX_LINK_SUB: v = __dsub_rn(a, b); break;
        case DLX_LINK_MUL: v = __dmul_rn(a, b); break;
        case DLX_LINK_DIV: v = __ddiv_rn(a, b); break;
        case DLX_LINK_ABS: v = fabs(a); break;
        case DLX_LINK_EXP: v = exp(a); break;
        default: v = __dsqrt_rn(a); break;
      }
      r[c.dst[q]] = v;
    }
    return r[c.out];
  }
};

template <int M, class Link, bool WRITE_H, class T = double>   // T: fp64 or fp32 storage of x
__global__ void __launch_bounds__(kRowThreads, DLX_ROW_MINB)
logreg_grad_kernel(const T* __restrict__ x, const long long* __restrict__ y, int64_t n,
                   int d, const double* __restrict__ theta, Link link, double* __restrict__ h_out,
                   double* __restrict__ parts) {
  pdl_wait();   // programmatic dependent launch: inputs are final from here on
  pdl_trigger();
  extern __shared__ double red_s[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double th[M][2], acc[M][2];
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const int j = 64 * m + 2 * lane;
    th[m][0] = j < d ? theta[j] : 0.0;
    th[m][1] = j + 1 < d ? theta[j + 1] : 0.0;
    acc[m][0] = acc[m][1] = 0.0;
  }
  // G blocks of 8 rows per warp step: fp32 storage keeps 16 rows (packed) in flight, the same
  // registers and bytes in flight as 8 fp64 rows (d <= 64; wider rows keep 8).  A warp's blocks
  // are w, w + W, w + 2W, ... either way, so the accumulation order (and every bit of the
  // result) is that of the fp64 kernel on the promoted matrix.
  constexpr int G = (sizeof(T) == 4 && M == 1) ? DLX_F32_GROUPS : 1;
  const int64_t nblk = (n + kRows - 1) / kRows;
  const int64_t W = static_cast<int64_t>(gridDim.x) * kRowWarps;
  const int my_row = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
  for (int64_t blk = static_cast<int64_t>(blockIdx.x) * kRowWarps + warp; blk < nblk; blk += G * W) {
    typename Vec2<T>::type v[G][kRows][M];
#pragma unroll
    for (int g = 0; g < G; ++g) load_rows<M>(x, (blk + g * W) * kRows, n, d, lane, v[g]);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (g > 0 && blk + g * W >= nblk) break;   // warp-uniform
      const int64_t i0 = (blk + g * W) * kRows;
      const int64_t iy = i0 + my_row;
      const double yv = iy < n ? static_cast<double>(__ldg(y + iy)) : 0.0;
      double2 e[kRows][M];   // promoted once (fp32 storage), used by the dot and the gradient
#pragma unroll
      for (int r = 0; r < kRows; ++r)
#pragma unroll
        for (int m = 0; m < M; ++m) e[r][m] = to_d2(v[g][r][m]);
      double p[kRows];
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        double a = 0.0;
#pragma unroll
        for (int m = 0; m < M; ++m) a = fma(th[m][0], e[r][m].x, fma(th[m][1], e[r][m].y, a));
        p[r] = a;
      }
      const double z = reduce_scatter8(p, lane);
      const double h = iy < n ? link(z) : 0.0;
      if (WRITE_H && (lane & 3) == 0 && iy < n) h_out[iy] = h;
      const double res = iy < n ? h - yv : 0.0;
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        const double rr = __shfl_sync(0xffffffffu, res, lane_of_row(r));
#pragma unroll
        for (int m = 0; m < M; ++m) {
          acc[m][0] = fma(rr, e[r][m].x, acc[m][0]);
          acc[m][1] = fma(rr, e[r][m].y, acc[m][1]);
        }
      }
    }
  }
  cta_reduce_columns<M>(acc, d, red_s, parts + static_cast<size_t>(blockIdx.x) * d);
}

// ---------------------------------------------------------------------------------------
// Bucket row sums — the keyed multi-sum multiloop (GDA pass 1: 1 + 2d reduces predicated on
// y(i) == c, loops.cpp:111-174): for the pass's KB bucket values b_t,
//   counts[t] = #{i : key_i == b_t},   sums[t][j] = sum_{key_i == b_t} x_ij.
// Same streaming skeleton as the gradient: a warp holds 8 rows, lane l columns {2l, 2l+1} + 64m;
// the key of each row is broadcast from lane r, and every bucket's accumulator adds the element
// only where the key matches (a select, not a 0/1 weight: 0 * inf would be NaN, and the
// reference adds nothing for a filtered-out index, loops.hpp:22-24).
struct Buckets {
  long long b[8];
};

template <int M, int KB, bool VEC>
__global__ void __launch_bounds__(kRowThreads, DLX_ROW_MINB)
bucket_rowsum_kernel(const double* __restrict__ x, const long long* __restrict__ key, int64_t n, int d,
                     Buckets bk, int nb, double* __restrict__ parts, long long* __restrict__ parts_cnt) {
  pdl_wait();   // programmatic dependent launch: inputs are final from here on
  pdl_trigger();
  extern __shared__ double red_s[];
  __shared__ long long cnt_s[kRowWarps][KB];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[KB][M][2];
  unsigned cnt[KB];   // rows a warp visits: < 2^32
#pragma unroll
  for (int t = 0; t < KB; ++t) {
    cnt[t] = 0;
#pragma unroll
    for (int m = 0; m < M; ++m) acc[t][m][0] = acc[t][m][1] = 0.0;
  }
  const int64_t nblk = (n + kRows - 1) / kRows;
  const int64_t W = static_cast<int64_t>(gridDim.x) * kRowWarps;
  for (int64_t blk = static_cast<int64_t>(blockIdx.x) * kRowWarps + warp; blk < nblk; blk += W) {
    const int64_t i0 = blk * kRows;
    double2 v[kRows][M];
    if (VEC) {
      load_rows<M>(x, i0, n, d, lane, v);
    } else {   // odd d: rows are not 16-byte aligned
#pragma unroll
      for (int r = 0; r < kRows; ++r)
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const int64_t i = i0 + r;
          const int j = 64 * m + 2 * lane;
          v[r][m].x = (i < n && j < d) ? __ldg(x + i * d + j) : 0.0;
          v[r][m].y = (i < n && j + 1 < d) ? __ldg(x + i * d + j + 1) : 0.0;
        }
    }
    const long long klane = (lane < kRows && i0 + lane < n) ? __ldg(key + i0 + lane) : 0;
    const bool live = lane < kRows && i0 + lane < n;
#pragma unroll
    for (int r = 0; r < kRows; ++r) {
      const long long kv = __shfl_sync(0xffffffffu, klane, r);
      const bool lv = __shfl_sync(0xffffffffu, live, r);
#pragma unroll
      for (int t = 0; t < KB; ++t) {
        const bool hit = lv && kv == bk.b[t];
        cnt[t] += hit;
#pragma unroll
        for (int m = 0; m < M; ++m) {
          acc[t][m][0] = hit ? acc[t][m][0] + v[r][m].x : acc[t][m][0];
          acc[t][m][1] = hit ? acc[t][m][1] + v[r][m].y : acc[t][m][1];
        }
      }
    }
  }
  if (lane == 0)   // every lane counted the same rows
#pragma unroll
    for (int t = 0; t < KB; ++t) cnt_s[warp][t] = cnt[t];
  // partial record of this CTA: nb (<= KB, the pass's real buckets) rows of d sums, nb counts
#pragma unroll
  for (int t = 0; t < KB; ++t)
    if (t < nb) cta_reduce_columns<M>(acc[t], d, red_s, parts + (static_cast<size_t>(blockIdx.x) * nb + t) * d);
  if (threadIdx.x < nb) {
    long long s = 0;
    for (int w = 0; w < kRowWarps; ++w) s += cnt_s[w][threadIdx.x];
    parts_cnt[static_cast<size_t>(blockIdx.x) * nb + threadIdx.x] = s;
  }
}

__global__ void gda_means_kernel(const long long* __restrict__ n1p, const double* __restrict__ s0,
                                 const double* __restrict__ s1, long long n_total, int d,
                                 double* __restrict__ mu0, double* __restrict__ mu1) {
  pdl_wait();   // programmatic dependent launch: inputs are final from here on
  pdl_trigger();
  const long long n1 = *n1p;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < d; j += gridDim.x * blockDim.x) {
    mu0[j] = s0[j] / static_cast<double>(n_total - n1);
    mu1[j] = s1[j] / static_cast<double>(n1);
  }
}

// ---------------------------------------------------------------------------------------
// GDA pass 2: S[a][b] = sum_i (x_ia - mu_{y_i,a}) (x_ib - mu_{y_i,b}).
// CTA tile of kTs centred rows in shared memory; the 16x16 thread grid owns B x B output
// blocks (register tiles), one fp64 FMA per (sample, cell).
constexpr int kTs = 32;

template <int B>
__global__ void __launch_bounds__(kRowThreads)
gda_pass2_kernel(const double* __restrict__ x, const long long* __restrict__ y, int64_t n, int d,
                 const double* __restrict__ mu0, const double* __restrict__ mu1,
                 double* __restrict__ parts) {
  pdl_wait();   // programmatic dependent launch: inputs are final from here on
  pdl_trigger();
  extern __shared__ double sm[];
  const int D = 16 * B;           // padded dimension
  double* mu_s = sm;              // 2 * D
  double* diff_s = sm + 2 * D;    // kTs * D
  const int tid = threadIdx.x;
  for (int j = tid; j < 2 * D; j += kRowThreads) {
    const int c = j / D, jj = j - c * D;
    mu_s[j] = jj < d ? (c ? mu1[jj] : mu0[jj]) : 0.0;
  }
  const int ta = tid >> 4, tb = tid & 15;
  double acc[B][B];
#pragma unroll
  for (int u = 0; u < B; ++u)
#pragma unroll
    for (int v = 0; v < B; ++v) acc[u][v] = 0.0;
  const int64_t ntiles = (n + kTs - 1) / kTs;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t i0 = t * kTs;
    __syncthreads();
    for (int e = tid; e < kTs * D; e += kRowThreads) {
      const int r = e / D, j = e - r * D;
      const int64_t i = i0 + r;
      double v = 0.0;
      if (i < n && j < d) {
        const long long yy = __ldg(y + i);
        v = __ldg(x + i * d + j) - mu_s[(yy == 1 ? D : 0) + j];
      }
      diff_s[r * D + j] = v;
    }
    __syncthreads();
#pragma unroll 4
    for (int r = 0; r < kTs; ++r) {
      double da[B], db[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        da[u] = diff_s[r * D + ta * B + u];
        db[u] = diff_s[r * D + tb * B + u];
      }
#pragma unroll
      for (int u = 0; u < B; ++u)
#pragma unroll
        for (int v = 0; v < B; ++v) acc[u][v] = fma(da[u], db[v], acc[u][v]);
    }
  }
  double* out = parts + static_cast<size_t>(blockIdx.x) * d * d;
#pragma unroll
  for (int u = 0; u < B; ++u)
#pragma unroll
    for (int v = 0; v < B; ++v) {
      const int a = ta * B + u, b = tb * B + v;
      if (a < d && b < d) out[a * d + b] = acc[u][v];
    }
}

}  // namespace dlx

namespace dlx {
int gda_pass2_dmma_grid(int64_t n);
int gda_pass2_dmma(const double* x, const long long* y, int64_t n, int d, const double* mu0,
                   const double* mu1, double* parts, size_t parts_bytes, double* out,
                   cudaStream_t stream);
}  // namespace dlx

using namespace dlx;

namespace {

int m_for(int d) { return (d + 63) / 64; }

int gda2_grid(int64_t n) {
  int64_t grid = static_cast<int64_t>(sm_count()) * 2;
  const int64_t tiles = (n + kTs - 1) / kTs;
  return static_cast<int>(std::max<int64_t>(1, std::min(grid, tiles)));
}

int gda2_b(int d) {
  if (d <= 16) return 1;
  if (d <= 32) return 2;
  if (d <= 64) return 4;
  if (d <= 128) return 8;
  return 0;
}

}  // namespace

extern "C" {

size_t dlx_logreg_workspace_bytes(int64_t n, int32_t d) {
  return static_cast<size_t>(row_grid(n)) * d * sizeof(double) + 256;
}

}  // extern "C"

template <class T>
static int logreg_grad_impl(const T* d_x, const int64_t* d_y, int64_t n, int32_t d, const double* d_theta,
                            double* d_grad, void* d_workspace, size_t workspace_bytes, dlx_stream_t stream) {
  DLX_REQUIRE(n >= 0 && d > 0, DLX_ERR_ARG, "logreg: bad shape");
  DLX_REQUIRE(d % 2 == 0 && m_for(d) <= kMaxM, DLX_ERR_GENERATION,
              "GenerationFailed: logreg needs even d <= %d (got %d)", 64 * kMaxM, d);
  const int grid = row_grid(n);
  const size_t need = static_cast<size_t>(grid) * d * sizeof(double);
  DLX_REQUIRE(d_workspace && workspace_bytes >= need, DLX_ERR_ARG, "logreg: workspace too small");
  double* parts = static_cast<double*>(d_workspace);
  const size_t smem = static_cast<size_t>(kRowWarps) * d * sizeof(double);
  const long long* y = reinterpret_cast<const long long*>(d_y);
  const SigmoidLink sig;
  switch (m_for(d)) {
    case 1: DLX_CUDA(launch_pdl(logreg_grad_kernel<1, SigmoidLink, false, T>, dim3(grid), dim3(kRowThreads), smem, stream, d_x, y, n, d, d_theta, sig, nullptr, parts)); break;
    case 2: DLX_CUDA(launch_pdl(logreg_grad_kernel<2, SigmoidLink, false, T>, dim3(grid), dim3(kRowThreads), smem, stream, d_x, y, n, d, d_theta, sig, nullptr, parts)); break;
    case 3: DLX_CUDA(launch_pdl(logreg_grad_kernel<3, SigmoidLink, false, T>, dim3(grid), dim3(kRowThreads), smem, stream, d_x, y, n, d, d_theta, sig, nullptr, parts)); break;
    default: DLX_CUDA(launch_pdl(logreg_grad_kernel<4, SigmoidLink, false, T>, dim3(grid), dim3(kRowThreads), smem, stream, d_x, y, n, d, d_theta, sig, nullptr, parts)); break;
  }
  DLX_LAUNCHED("logreg_grad_kernel");
  return combine_f64(parts, grid, d, d_grad, stream);
}

extern "C" {

int dlx_logreg_grad(const double* d_x, const int64_t* d_y, int64_t n, int32_t d,
                    const double* d_theta, double* d_grad, void* d_workspace,
                    size_t workspace_bytes, dlx_stream_t stream) {
  return logreg_grad_impl(d_x, d_y, n, d, d_theta, d_grad, d_workspace, workspace_bytes, stream);
}

int dlx_logreg_grad_f32(const float* d_x, const int64_t* d_y, int64_t n, int32_t d,
                        const double* d_theta, double* d_grad, void* d_workspace,
                        size_t workspace_bytes, dlx_stream_t stream) {
  return logreg_grad_impl(d_x, d_y, n, d, d_theta, d_grad, d_workspace, workspace_bytes, stream);
}

int dlx_link_kind(const dlx_link_code* h_link) { return h_link ? static_cast<int>(link_kind(*h_link)) : -1; }

int dlx_rowdot_link_grad(const double* d_x, const int64_t* d_y, int64_t n, int32_t d, const double* d_theta,
                         const dlx_link_code* h_link, double* d_h, double* d_grad, void* d_workspace,
                         size_t workspace_bytes, dlx_stream_t stream) {
  DLX_REQUIRE(n >= 0 && d > 0 && h_link, DLX_ERR_ARG, "rowdot_link_grad: bad arguments");
  DLX_REQUIRE(h_link->n >= 0 && h_link->n <= DLX_LINK_MAX_CODE && h_link->out >= 0 && h_link->out < DLX_LINK_MAX_REGS,
              DLX_ERR_ARG, "rowdot_link_grad: bad link code");
  for (int q = 0; q < h_link->n; ++q)
    DLX_REQUIRE(h_link->dst[q] < DLX_LINK_MAX_REGS && h_link->a[q] < DLX_LINK_MAX_REGS && h_link->b[q] < DLX_LINK_MAX_REGS &&
                h_link->op[q] <= DLX_LINK_SQRT, DLX_ERR_ARG, "rowdot_link_grad: bad link instruction %d", q);
  DLX_REQUIRE(d % 2 == 0 && m_for(d) <= kMaxM, DLX_ERR_GENERATION,
              "GenerationFailed: the row-dot gradient needs even d <= %d (got %d)", 64 * kMaxM, d);
  const int grid = row_grid(n);
  const size_t need = static_cast<size_t>(grid) * d * sizeof(double);
  DLX_REQUIRE(d_workspace && workspace_bytes >= need, DLX_ERR_ARG, "rowdot_link_grad: workspace too small");
  double* parts = static_cast<double*>(d_workspace);
  const size_t smem = static_cast<size_t>(kRowWarps) * d * sizeof(double);
  const long long* y = reinterpret_cast<const long long*>(d_y);
  const CodeLink code{*h_link};
  const LinkKind kind = getenv("DLX_LINK_INTERPRET") ? kLinkCode : link_kind(*h_link);
#define DLX_RDL_L(MM, L, LV)                                                                                        \
  (d_h ? launch_pdl(logreg_grad_kernel<MM, L, true>, dim3(grid), dim3(kRowThreads), smem, stream, d_x, y, n, d,   \
                    d_theta, LV, d_h, parts)                                                                      \
       : launch_pdl(logreg_grad_kernel<MM, L, false>, dim3(grid), dim3(kRowThreads), smem, stream, d_x, y, n, d,  \
                    d_theta, LV, nullptr, parts))
#define DLX_RDL(MM)                                                                    \
  (kind == kLinkSigmoid ? DLX_RDL_L(MM, SigmoidLink, SigmoidLink{})                    \
   : kind == kLinkSoftsign ? DLX_RDL_L(MM, SoftsignLink, SoftsignLink{})               \
                           : DLX_RDL_L(MM, CodeLink, code))
  switch (m_for(d)) {
    case 1: DLX_CUDA(DLX_RDL(1)); break;
    case 2: DLX_CUDA(DLX_RDL(2)); break;
    case 3: DLX_CUDA(DLX_RDL(3)); break;
    default: DLX_CUDA(DLX_RDL(4)); break;
  }
#undef DLX_RDL
#undef DLX_RDL_L
  DLX_LAUNCHED("logreg_grad_kernel");
  return combine_f64(parts, grid, d, d_grad, stream);
}

size_t dlx_gda_workspace_bytes(int64_t n, int32_t d) {
  const size_t p1 = dlx_bucket_rowsum_workspace_bytes(n, d, 2) + 2 * d * sizeof(double) + 1024;
  const size_t p2 = static_cast<size_t>(std::max(gda2_grid(n), gda_pass2_dmma_grid(n))) * d * d *
                        sizeof(double) + 256;
  return std::max(p1, p2);
}

}  // extern "C"

namespace {
// buckets per pass for a row of M column groups (registers: KB * M * 2 accumulators per lane)
int buckets_per_pass(int M) { return M == 1 ? 4 : M == 2 ? 2 : 1; }

template <int M, int KB>
int launch_bucket_rowsum(bool vec, dim3 grid, size_t smem, cudaStream_t stream, const double* x,
                         const long long* key, int64_t n, int d, const Buckets& bk, int nb, double* parts,
                         long long* pc) {
  if (vec)
    DLX_CUDA(launch_pdl(bucket_rowsum_kernel<M, KB, true>, grid, dim3(kRowThreads), smem, stream, x, key, n, d, bk, nb, parts, pc));
  else
    DLX_CUDA(launch_pdl(bucket_rowsum_kernel<M, KB, false>, grid, dim3(kRowThreads), smem, stream, x, key, n, d, bk, nb, parts, pc));
  DLX_LAUNCHED("bucket_rowsum_kernel");
  return DLX_OK;
}
}  // namespace

extern "C" {

size_t dlx_bucket_rowsum_workspace_bytes(int64_t n, int32_t d, int32_t nbuckets) {
  (void)nbuckets;
  return static_cast<size_t>(row_grid(n)) * 4 * (static_cast<size_t>(std::max(d, 1)) * sizeof(double) + sizeof(long long)) + 1024;
}

int dlx_bucket_rowsum(const double* d_x, const int64_t* d_keys, int64_t n, int32_t d,
                      const int64_t* h_buckets, int32_t nbuckets, int64_t* d_counts, double* d_sums,
                      void* d_workspace, size_t workspace_bytes, dlx_stream_t stream) {
  DLX_REQUIRE(n >= 0 && d > 0 && nbuckets >= 0 && (nbuckets == 0 || h_buckets), DLX_ERR_ARG, "bucket_rowsum: bad arguments");
  DLX_REQUIRE(m_for(d) <= kMaxM, DLX_ERR_GENERATION,
              "GenerationFailed: bucket row sums need d <= %d (got %d)", 64 * kMaxM, d);
  const int M = m_for(d) == 3 ? 4 : m_for(d);
  const int KB = (M == 1 && nbuckets <= 2) ? 2 : buckets_per_pass(M);   // GDA's two classes: KB = 2
  const int grid = row_grid(n);
  Carve c(d_workspace);
  double* parts = c.take<double>(static_cast<size_t>(grid) * KB * d);
  long long* pc = c.take<long long>(static_cast<size_t>(grid) * KB);
  DLX_REQUIRE(d_workspace && c.used <= workspace_bytes, DLX_ERR_ARG, "bucket_rowsum: workspace too small");
  const size_t smem = static_cast<size_t>(kRowWarps) * d * sizeof(double);
  const long long* key = reinterpret_cast<const long long*>(d_keys);
  const bool vec = d % 2 == 0;
  for (int b0 = 0; b0 < nbuckets; b0 += KB) {   // one pass over x per KB buckets
    Buckets bk;
    const int nb = std::min(KB, nbuckets - b0);
    for (int t = 0; t < 8; ++t) bk.b[t] = t < nb ? h_buckets[b0 + t] : (t > 0 ? bk.b[t - 1] : 0);
    int rc;
    switch (M) {
      case 1: rc = KB == 2 ? launch_bucket_rowsum<1, 2>(vec, dim3(grid), smem, stream, d_x, key, n, d, bk, nb, parts, pc)
                           : launch_bucket_rowsum<1, 4>(vec, dim3(grid), smem, stream, d_x, key, n, d, bk, nb, parts, pc); break;
      case 2: rc = launch_bucket_rowsum<2, 2>(vec, dim3(grid), smem, stream, d_x, key, n, d, bk, nb, parts, pc); break;
      default: rc = launch_bucket_rowsum<4, 1>(vec, dim3(grid), smem, stream, d_x, key, n, d, bk, nb, parts, pc); break;
    }
    if (rc != DLX_OK) return rc;
    // padding buckets (t >= nb) repeat the last value and are not written
    rc = combine_f64_i64(parts, static_cast<long long>(nb) * d, d_sums + static_cast<size_t>(b0) * d, pc, nb,
                         reinterpret_cast<long long*>(d_counts) + b0, grid, stream);
    if (rc != DLX_OK) return rc;
    if (nb < KB) break;
  }
  return DLX_OK;
}

int dlx_gda_pass1(const double* d_x, const int64_t* d_y, int64_t n, int32_t d, int64_t* d_n1,
                  double* d_sum0, double* d_sum1, void* d_workspace, size_t workspace_bytes,
                  dlx_stream_t stream) {
  // classes 0 and 1 as buckets: sums land contiguously (class 0 then class 1) in a scratch
  // record carved after the row partials
  DLX_REQUIRE(n >= 0 && d > 0, DLX_ERR_ARG, "gda: bad shape");
  DLX_REQUIRE(d % 2 == 0 && m_for(d) <= kMaxM, DLX_ERR_GENERATION,
              "GenerationFailed: gda needs even d <= %d (got %d)", 64 * kMaxM, d);
  const size_t need = dlx_bucket_rowsum_workspace_bytes(n, d, 2);
  Carve c(d_workspace);
  c.take<char>(need);
  double* sums = c.take<double>(2 * static_cast<size_t>(d));
  long long* cnt = c.take<long long>(2);
  DLX_REQUIRE(d_workspace && c.used <= workspace_bytes, DLX_ERR_ARG, "gda: workspace too small");
  const int64_t classes[2] = {0, 1};
  int rc = dlx_bucket_rowsum(d_x, d_y, n, d, classes, 2, reinterpret_cast<int64_t*>(cnt), sums, d_workspace,
                             need, stream);
  if (rc != DLX_OK) return rc;
  DLX_CUDA(cudaMemcpyAsync(d_sum0, sums, d * sizeof(double), cudaMemcpyDeviceToDevice, stream));
  DLX_CUDA(cudaMemcpyAsync(d_sum1, sums + d, d * sizeof(double), cudaMemcpyDeviceToDevice, stream));
  DLX_CUDA(cudaMemcpyAsync(d_n1, cnt + 1, sizeof(long long), cudaMemcpyDeviceToDevice, stream));
  return DLX_OK;
}

int dlx_gda_means(const int64_t* d_n1, const double* d_sum0, const double* d_sum1,
                  int64_t n_total, int32_t d, double* d_mu0, double* d_mu1, dlx_stream_t stream) {
  DLX_REQUIRE(d > 0, DLX_ERR_ARG, "gda means: bad d");
  DLX_CUDA(launch_pdl(gda_means_kernel, dim3((d + 127) / 128), dim3(128), 0, stream, 
      reinterpret_cast<const long long*>(d_n1), d_sum0, d_sum1, n_total, d, d_mu0, d_mu1));
  DLX_LAUNCHED("gda_means_kernel");
  return DLX_OK;
}

int dlx_gda_pass2(const double* d_x, const int64_t* d_y, int64_t n, int32_t d,
                  const double* d_mu0, const double* d_mu1, double* d_scatter, void* d_workspace,
                  size_t workspace_bytes, dlx_stream_t stream) {
  DLX_REQUIRE(n >= 0 && d > 0, DLX_ERR_ARG, "gda: bad shape");
  if (d <= 64)  // fp64 tensor-core (DMMA) scatter
    return gda_pass2_dmma(d_x, reinterpret_cast<const long long*>(d_y), n, d, d_mu0, d_mu1,
                          static_cast<double*>(d_workspace), workspace_bytes, d_scatter, stream);
  const int B = gda2_b(d);
  DLX_REQUIRE(B > 0, DLX_ERR_GENERATION, "GenerationFailed: gda pass 2 needs d <= 128 (got %d)", d);
  const int grid = gda2_grid(n);
  const size_t need = static_cast<size_t>(grid) * d * d * sizeof(double);
  DLX_REQUIRE(d_workspace && workspace_bytes >= need, DLX_ERR_ARG, "gda: workspace too small");
  double* parts = static_cast<double*>(d_workspace);
  const size_t smem = static_cast<size_t>(2 + kTs) * 16 * B * sizeof(double);
  const long long* y = reinterpret_cast<const long long*>(d_y);
  switch (B) {
    case 1: DLX_CUDA(launch_pdl(gda_pass2_kernel<1>, dim3(grid), dim3(kRowThreads), smem, stream, d_x, y, n, d, d_mu0, d_mu1, parts)); break;
    case 2: DLX_CUDA(launch_pdl(gda_pass2_kernel<2>, dim3(grid), dim3(kRowThreads), smem, stream, d_x, y, n, d, d_mu0, d_mu1, parts)); break;
    case 4: DLX_CUDA(launch_pdl(gda_pass2_kernel<4>, dim3(grid), dim3(kRowThreads), smem, stream, d_x, y, n, d, d_mu0, d_mu1, parts)); break;
    default: DLX_CUDA(launch_pdl(gda_pass2_kernel<8>, dim3(grid), dim3(kRowThreads), smem, stream, d_x, y, n, d, d_mu0, d_mu1, parts)); break;
  }
  DLX_LAUNCHED("gda_pass2_kernel");
  return combine_f64(parts, grid, static_cast<long long>(d) * d, d_scatter, stream);
}

int dlx_axpy_inplace(double* d_theta, const double* d_grad, double alpha, int64_t n,
                     dlx_stream_t stream);

}  // extern "C"
