// gda_dmma.cu — GDA pass 2: the scatter S = sum_i (x_i - mu_{y_i})(x_i -
// mu_{y_i})^T as a dense contraction on the fp64 tensor cores.
//
// The reference computes it as d*d separate reduce elems (one per (a, b) cell) over the same
// index traversal; here the centred rows of a 128-sample tile are staged in shared memory and
// each 8x8 output block is accumulated with mma.sync m8n8k4 f64 (SASS DMMA): fp64 products
// and fp64 accumulation, so the only difference from the reference is summation order (rtol
// 1e-9 is the stated tolerance).  S is symmetric: only the (d/8)(d/8+1)/2 lower blocks are
// accumulated and mirrored on output (the reference's S[a][b] and S[b][a] are bit-identical
// too, both being the same ordered sum of identical products).
#include <algorithm>

#include "common.cuh"

namespace dlx {

constexpr int kGdThreads = 256;
constexpr int kGdWarps = kGdThreads / 32;
constexpr int kGdTile = 128;          // samples per staged tile
constexpr int kGdStride = 64 + 4;     // padded row stride (doubles): 2-way max on 8-byte loads
constexpr int kGdMaxBlocksPerWarp = 5;  // 36 lower blocks of a 64x64 S over 8 warps

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(kGdThreads, 3)
gda_pass2_dmma_kernel(const double* __restrict__ x, const long long* __restrict__ y, int64_t n,
                      int d, const double* __restrict__ mu0, const double* __restrict__ mu1,
                      double* __restrict__ parts) {
  pdl_wait();   // programmatic dependent launch: inputs are final from here on
  pdl_trigger();
  __shared__ double mu_s[2][64];
  extern __shared__ double diff_s[];  // [kGdTile][kGdStride]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = (d + 7) / 8;                 // 8-wide blocks per side
  const int nblocks = nb * (nb + 1) / 2;      // lower-triangular blocks
  for (int j = tid; j < 128; j += kGdThreads) {
    const int c = j >> 6, jj = j & 63;
    mu_s[c][jj] = jj < d ? (c ? mu1[jj] : mu0[jj]) : 0.0;
  }
  // blocks owned by this warp: t = warp + 8u, decoded to (ba >= bb)
  int ba[kGdMaxBlocksPerWarp], bb[kGdMaxBlocksPerWarp];
  double acc[kGdMaxBlocksPerWarp][2];
#pragma unroll
  for (int u = 0; u < kGdMaxBlocksPerWarp; ++u) {
    int t = warp + kGdWarps * u;
    int a = 0;
    while (t >= a + 1) { t -= a + 1; ++a; }
    ba[u] = a;
    bb[u] = t;
    acc[u][0] = acc[u][1] = 0.0;
  }
  const int g = lane >> 2, kq = lane & 3;
  const int64_t ntiles = (n + kGdTile - 1) / kGdTile;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i0 = tile * kGdTile;
    __syncthreads();
    // stage centred rows: diff[s][j] = x[i0+s][j] - mu_{y}[j]  (zero outside n / d)
    // 8 independent loads per thread in flight before their stores (a load -> store loop
    // would expose the full memory latency per element)
    for (int e0 = tid; e0 < kGdTile * 64; e0 += 8 * kGdThreads) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * kGdThreads;
        const int s = e >> 6, j = e & 63;
        const int64_t i = i0 + s;
        v[u] = 0.0;
        if (i < n && j < d) v[u] = __ldg(x + i * d + j) - mu_s[__ldg(y + i) == 1 ? 1 : 0][j];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * kGdThreads;
        diff_s[(e >> 6) * kGdStride + (e & 63)] = v[u];
      }
    }
    __syncthreads();
#pragma unroll 2
    for (int k0 = 0; k0 < kGdTile; k0 += 4) {
      const double* row = diff_s + (k0 + kq) * kGdStride;
#pragma unroll
      for (int u = 0; u < kGdMaxBlocksPerWarp; ++u) {
        if (warp + kGdWarps * u < nblocks) {
          const double a = row[ba[u] * 8 + g];   // A[r=g][k=kq] = diff[k0+kq][8*ba + g]
          const double b = row[bb[u] * 8 + g];   // B[k=kq][c=g] = diff[k0+kq][8*bb + g]
          dmma_8x8x4(acc[u], a, b);
        }
      }
    }
  }
  // C[r][c]: r = g, c = 2*kq + {0,1}; write block and its mirror
  double* out = parts + static_cast<size_t>(blockIdx.x) * d * d;
#pragma unroll
  for (int u = 0; u < kGdMaxBlocksPerWarp; ++u) {
    if (warp + kGdWarps * u >= nblocks) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = ba[u] * 8 + g, c = bb[u] * 8 + 2 * kq + h;
      if (r < d && c < d) {
        out[r * d + c] = acc[u][h];
        if (ba[u] != bb[u]) out[c * d + r] = acc[u][h];
      }
    }
  }
}

int gda_pass2_dmma_grid(int64_t n) {
  const int64_t tiles = (n + kGdTile - 1) / kGdTile;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(tiles, sm_count() * 3)));
}

int gda_pass2_dmma(const double* x, const long long* y, int64_t n, int d, const double* mu0,
                   const double* mu1, double* parts, size_t parts_bytes, double* out,
                   cudaStream_t stream) {
  DLX_REQUIRE(d <= 64, DLX_ERR_GENERATION, "GenerationFailed: DMMA scatter plan needs d <= 64");
  const int grid = gda_pass2_dmma_grid(n);
  DLX_REQUIRE(parts && parts_bytes >= static_cast<size_t>(grid) * d * d * sizeof(double),
              DLX_ERR_ARG, "gda: workspace too small");
  const size_t smem = static_cast<size_t>(kGdTile) * kGdStride * sizeof(double);
  DLX_CUDA(cudaFuncSetAttribute(gda_pass2_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
  DLX_CUDA(launch_pdl(gda_pass2_dmma_kernel, dim3(grid), dim3(kGdThreads), smem, stream, x, y, n, d, mu0, mu1, parts));
  DLX_LAUNCHED("gda_pass2_dmma_kernel");
  return combine_f64(parts, grid, static_cast<long long>(d) * d, out, stream);
}

}  // namespace dlx
