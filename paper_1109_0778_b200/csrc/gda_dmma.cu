// gda_dmma.cu — GDA pass 2: the scatter S = sum_i (x_i - mu_{y_i})(x_i -
// mu_{y_i})^T as a dense contraction on the fp64 tensor cores.
//
// The reference computes it as d*d separate reduce elems (one per (a, b) cell) over the same
// index traversal; here 128-sample tiles are centred in shared memory and each 8x8 output
// block is accumulated with mma.sync m8n8k4 f64 (SASS DMMA): fp64 products and fp64
// accumulation, so the only difference from the reference is summation order (rtol 1e-9 is
// the stated tolerance).  S is symmetric: only the (d/8)(d/8+1)/2 lower blocks are
// accumulated and mirrored on output (the reference's S[a][b] and S[b][a] are bit-identical
// too, both being the same ordered sum of identical products).
//
// Data movement: one persistent CTA per SM, warp-specialised.  Each 64-sample tile's raw rows
// (64 x d fp64, contiguous in the row-major matrix) and labels arrive by 1-D bulk TMA copies
// into a three-slot ring, issued three tiles ahead, so HBM latency never stalls a warp (the
// previous version's long-scoreboard stalls).  Eight centring warps turn a raw slot into a
// padded operand tile D[b] = x - mu_y (row stride 68 doubles: the fragment loads of four
// consecutive rows fall in distinct banks; two D buffers, mbarrier full/empty handshakes)
// while twelve tensor-core warps own 3 lower blocks each (36 = 12 x 3 for d = 64) and run the
// DMMA chains on the other D buffer, so centring overlaps the tensor-core phase.  (With four
// centring warps the tensor-core warps sat on empty D buffers 20% of the time, profile r73.)
#include <algorithm>

#include "common.cuh"
#include "sm100.cuh"

namespace dlx {

using namespace sm100;

constexpr int kGdMmaWarps = 12;                     // tensor-core warps: 3 lower blocks each
#ifndef DLX_GDA_CTR_WARPS
#define DLX_GDA_CTR_WARPS 8
#endif
#ifndef DLX_GDA_DBUFS
#define DLX_GDA_DBUFS 2
#endif
constexpr int kGdCtrWarps = DLX_GDA_CTR_WARPS;      // centring warps (two per SM sub-partition)
constexpr int kGdThreads = (kGdMmaWarps + kGdCtrWarps) * 32;
constexpr int kGdCtrThreads = kGdCtrWarps * 32;
constexpr int kGdTile = 64;           // samples per tile
constexpr int kGdStride = 64 + 4;     // padded operand row stride (doubles)
constexpr int kGdBlocksPerWarp = 3;   // 36 lower blocks of a 64x64 S over 12 warps
constexpr int kGdSlots = 3;           // raw tile ring (bulk copies in flight)
constexpr int kGdDBufs = DLX_GDA_DBUFS;   // centred operand tiles
constexpr size_t kGdRawBytes = static_cast<size_t>(kGdTile) * 64 * 8;
constexpr size_t kGdDBytes = static_cast<size_t>(kGdTile) * kGdStride * 8;
constexpr size_t kGdOffY = kGdSlots * kGdRawBytes;
constexpr size_t kGdOffD = kGdOffY + kGdSlots * kGdTile * 8;
constexpr size_t kGdOffMu = kGdOffD + kGdDBufs * kGdDBytes;
constexpr size_t kGdOffBar = kGdOffMu + 2 * 64 * 8;
constexpr size_t kGdSmem = kGdOffBar + (kGdSlots + 2 * kGdDBufs) * 8;

// d = 64: the 36 lower 8x8 blocks as 12 triples {si, o0, o1, o2} = blocks (si, o_u) sharing the
// index si (each unordered pair {a, b} with a >= b appears once)
__constant__ int kGdTriples[kGdMmaWarps][4] = {
    {0, 0, 2, 3}, {0, 4, 5, 7}, {1, 0, 1, 2}, {1, 4, 5, 6}, {2, 2, 3, 4}, {2, 5, 6, 7},
    {3, 1, 3, 4}, {3, 5, 6, 7}, {4, 4, 5, 6}, {5, 5, 6, 7}, {6, 0, 6, 7}, {7, 1, 4, 7}};

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(kGdThreads, 1)
gda_pass2_dmma_kernel(const double* __restrict__ x, const long long* __restrict__ y, int64_t n,
                      int d, const double* __restrict__ mu0, const double* __restrict__ mu1,
                      double* __restrict__ parts) {
  extern __shared__ __align__(1024) unsigned char smem[];
  double* const raw = reinterpret_cast<double*>(smem);
  long long* const ys = reinterpret_cast<long long*>(smem + kGdOffY);
  double* const Dbuf = reinterpret_cast<double*>(smem + kGdOffD);
  double* const mu_s = reinterpret_cast<double*>(smem + kGdOffMu);   // [2][64]
  uint64_t* const raw_full = reinterpret_cast<uint64_t*>(smem + kGdOffBar);
  uint64_t* const d_full = raw_full + kGdSlots;
  uint64_t* const d_empty = d_full + kGdDBufs;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t ntiles = (n + kGdTile - 1) / kGdTile;
  const int mt = static_cast<int>(ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0);
  const bool bulk_ok = (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0;
  auto tile_of = [&](int m) { return static_cast<int64_t>(blockIdx.x) + static_cast<int64_t>(m) * gridDim.x; };
  auto full_tile = [&](int m) { return bulk_ok && (tile_of(m) + 1) * kGdTile <= n; };
  constexpr int kIssuer = kGdMmaWarps * 32;   // first centring thread issues the bulk copies
  auto issue = [&](int m) {   // tile m into raw slot m % 3 (a bare arrive for an edge tile)
    const int s = m % kGdSlots;
    const int64_t t = tile_of(m);
    if (full_tile(m)) {
      const uint32_t bx = static_cast<uint32_t>(kGdTile) * static_cast<uint32_t>(d) * 8u;
      mbar_arrive_expect_tx(&raw_full[s], bx + kGdTile * 8);
      bulk_g2s(raw + static_cast<size_t>(s) * kGdTile * 64, x + t * kGdTile * d, bx, &raw_full[s]);
      bulk_g2s(ys + s * kGdTile, y + t * kGdTile, kGdTile * 8, &raw_full[s]);
    } else {
      mbar_arrive(&raw_full[s]);   // the centring warps read this tile from global memory
    }
  };
  if (tid == 0) {
    for (int s = 0; s < kGdSlots; ++s) mbar_init(&raw_full[s], 1);
    for (int b = 0; b < kGdDBufs; ++b) {
      mbar_init(&d_full[b], 1);
      mbar_init(&d_empty[b], kGdMmaWarps);
    }
    fence_mbar_init();
  }
  // programmatic dependent launch: the predecessor may still be running until here (it may
  // even be the kernel that wrote x), so every global read comes after the wait
  pdl_wait();
  pdl_trigger();
  for (int j = tid; j < 128; j += kGdThreads) {
    const int c = j >> 6, jj = j & 63;
    mu_s[j] = jj < d ? (c ? mu1[jj] : mu0[jj]) : 0.0;
  }
  __syncthreads();

  if (warp >= kGdMmaWarps) {
    // ---- centring warps: raw slot -> D[b] = x - mu_y (zero outside n / d) -----------------
    const int ct = tid - kIssuer;
    if (ct == 0)
      for (int m = 0; m < kGdSlots && m < mt; ++m) issue(m);
    for (int m = 0; m < mt; ++m) {
      const int s = m % kGdSlots, b = m % kGdDBufs;
      const int64_t i0 = tile_of(m) * kGdTile;
      const int rows = static_cast<int>(std::min<int64_t>(kGdTile, n - i0));
      const bool from_smem = full_tile(m);
      mbar_wait(&raw_full[s], (m / kGdSlots) & 1);
      if (m >= kGdDBufs) mbar_wait(&d_empty[b], ((m - kGdDBufs) / kGdDBufs) & 1);
      const double* rs = raw + static_cast<size_t>(s) * kGdTile * 64;
      const long long* yv = ys + s * kGdTile;
      double* D = Dbuf + static_cast<size_t>(b) * kGdTile * kGdStride;
      if (from_smem && d == 64) {
        // fast path: thread = column pair (2cp, 2cp+1) x row phase; mu pair in registers, one
        // label broadcast per warp-row, 16-byte loads and stores
        const int cp = ct & 31, rp = ct >> 5;
        const double2 m0 = *reinterpret_cast<const double2*>(mu_s + 2 * cp);
        const double2 m1 = *reinterpret_cast<const double2*>(mu_s + 64 + 2 * cp);
#pragma unroll 4
        for (int r = rp; r < kGdTile; r += kGdCtrWarps) {
          const double2 xv = *reinterpret_cast<const double2*>(rs + r * 64 + 2 * cp);
          const bool one = yv[r] == 1;
          double2 o;
          o.x = xv.x - (one ? m1.x : m0.x);
          o.y = xv.y - (one ? m1.y : m0.y);
          *reinterpret_cast<double2*>(D + r * kGdStride + 2 * cp) = o;
        }
      } else
#pragma unroll 2
      for (int e0 = ct; e0 < kGdTile * 64; e0 += 4 * kGdCtrThreads) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int e = e0 + u * kGdCtrThreads;
          const int r = e >> 6, j = e & 63;
          v[u] = 0.0;
          if (r < rows && j < d) {
            const double xv = from_smem ? rs[r * d + j] : __ldg(x + (i0 + r) * d + j);
            const long long lab = from_smem ? yv[r] : __ldg(y + i0 + r);
            v[u] = xv - mu_s[(lab == 1 ? 64 : 0) + j];
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int e = e0 + u * kGdCtrThreads;
          D[(e >> 6) * kGdStride + (e & 63)] = v[u];
        }
      }
      named_bar(1, kGdCtrThreads);   // D[b] written, raw slot s read by every centring thread
      if (ct == 0) {
        mbar_arrive(&d_full[b]);
        if (m + kGdSlots < mt) {
          fence_proxy_async_smem();   // generic-proxy reads of slot s before the async refill
          issue(m + kGdSlots);
        }
      }
    }
    return;
  }

  // ---- tensor-core warps ----------------------------------------------------------------
  // d = 64: warp w owns blocks (si, o0), (si, o1), (si, o2) of kGdTriples[w] — every lower 8x8
  // block exactly once, three per warp sharing one index, so a k-step loads 4 fragments for 3
  // DMMAs (A and B fragments of an index are the same register: D[k0+kq][8*idx + g]).  Other d:
  // blocks t = warp + 12u of the lower triangle, 2 fragments per DMMA.
  const int nb = (d + 7) / 8;
  const int nblocks = nb * (nb + 1) / 2;
  const bool shared = nb == 8;
  int ba[kGdBlocksPerWarp], bb[kGdBlocksPerWarp];
  double acc[kGdBlocksPerWarp][2][2];   // [block][k-step parity][C pair]: 6 independent DMMA chains
#pragma unroll
  for (int u = 0; u < kGdBlocksPerWarp; ++u) {
    if (shared) {
      ba[u] = kGdTriples[warp][0];
      bb[u] = kGdTriples[warp][1 + u];
    } else {
      int t = warp + kGdMmaWarps * u;
      int a = 0;
      while (t >= a + 1) { t -= a + 1; ++a; }
      ba[u] = a;
      bb[u] = t;
    }
    acc[u][0][0] = acc[u][0][1] = acc[u][1][0] = acc[u][1][1] = 0.0;
  }
  const bool own[kGdBlocksPerWarp] = {shared || warp < nblocks, shared || warp + kGdMmaWarps < nblocks,
                                      shared || warp + 2 * kGdMmaWarps < nblocks};
  const int g = lane >> 2, kq = lane & 3;
  for (int m = 0; m < mt; ++m) {
    const int b = m % kGdDBufs;
    mbar_wait(&d_full[b], (m / kGdDBufs) & 1);
    const double* D = Dbuf + static_cast<size_t>(b) * kGdTile * kGdStride;
    if (shared) {
#pragma unroll 2
      for (int k0 = 0; k0 < kGdTile; k0 += 8) {
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const double* row = D + (k0 + 4 * p + kq) * kGdStride + g;
          const double fa = row[ba[0] * 8];
#pragma unroll
          for (int u = 0; u < kGdBlocksPerWarp; ++u) dmma_8x8x4(acc[u][p], fa, row[bb[u] * 8]);
        }
      }
    } else {
#pragma unroll 2
      for (int k0 = 0; k0 < kGdTile; k0 += 8) {
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const double* row = D + (k0 + 4 * p + kq) * kGdStride + g;
#pragma unroll
          for (int u = 0; u < kGdBlocksPerWarp; ++u)
            if (own[u]) dmma_8x8x4(acc[u][p], row[ba[u] * 8], row[bb[u] * 8]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&d_empty[b]);
  }
  // C[r][c] of block (ba, bb): r = g, c = 2*kq + {0,1}; write the block and its mirror
  double* out = parts + static_cast<size_t>(blockIdx.x) * d * d;
#pragma unroll
  for (int u = 0; u < kGdBlocksPerWarp; ++u) {
    if (!own[u]) continue;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = ba[u] * 8 + g, c = bb[u] * 8 + 2 * kq + h;
      if (r < d && c < d) {
        const double v = acc[u][0][h] + acc[u][1][h];
        out[r * d + c] = v;
        if (ba[u] != bb[u]) out[c * d + r] = v;
      }
    }
  }
}

int gda_pass2_dmma_grid(int64_t n) {
  const int64_t tiles = (n + kGdTile - 1) / kGdTile;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(tiles, sm_count())));
}

int gda_pass2_dmma(const double* x, const long long* y, int64_t n, int d, const double* mu0,
                   const double* mu1, double* parts, size_t parts_bytes, double* out,
                   cudaStream_t stream) {
  DLX_REQUIRE(d <= 64, DLX_ERR_GENERATION, "GenerationFailed: DMMA scatter plan needs d <= 64");
  const int grid = gda_pass2_dmma_grid(n);
  DLX_REQUIRE(parts && parts_bytes >= static_cast<size_t>(grid) * d * d * sizeof(double),
              DLX_ERR_ARG, "gda: workspace too small");
  DLX_CUDA(cudaFuncSetAttribute(gda_pass2_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kGdSmem)));
  DLX_CUDA(launch_pdl(gda_pass2_dmma_kernel, dim3(grid), dim3(kGdThreads), kGdSmem, stream, x, y, n, d, mu0, mu1, parts));
  DLX_LAUNCHED("gda_pass2_dmma_kernel");
  return combine_f64(parts, grid, static_cast<long long>(d) * d, out, stream);
}

}  // namespace dlx
