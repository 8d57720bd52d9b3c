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
// previous version's long-scoreboard stalls).  Twelve centring warps turn a raw slot into a
// padded operand tile D[b] = x - mu_y (row stride 68 doubles: the fragment loads of four
// consecutive rows fall in distinct banks; two D buffers, mbarrier full/empty handshakes)
// while twelve tensor-core warps own 3 lower blocks each (36 = 12 x 3 for d = 64) and run the
// DMMA chains on the other D buffer, so centring overlaps the tensor-core phase.  (With four
// centring warps the tensor-core warps sat on empty D buffers 20% of the time, profile r73;
// eight suffice for pass 2 alone, twelve keep up with the single-pass fit's class sums, r81.)
#include <cuda.h>

#include <algorithm>
#include <type_traits>
#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"

namespace dlx {

using namespace sm100;

constexpr int kGdMmaWarps = 12;                     // tensor-core warps: 3 lower blocks each
#ifndef DLX_GDA_CTR_WARPS
#define DLX_GDA_CTR_WARPS 12
#endif
#ifndef DLX_GDA_DBUFS
#define DLX_GDA_DBUFS 2
#endif
constexpr int kGdCtrWarps = DLX_GDA_CTR_WARPS;      // centring warps (three per SM sub-partition)
constexpr int kGdThreads = (kGdMmaWarps + kGdCtrWarps) * 32;
constexpr int kGdCtrThreads = kGdCtrWarps * 32;
constexpr int kGdTile = 64;           // samples per tile
// Operand tile layout: rows k and k + 4 of each 8-row group are interleaved per column, so one
// 16-byte load gives a lane its fragments for both k-steps of the group (pair-row pr = 4 * group
// + k % 4 holds [col][k / 4 % 2]); pair-row stride 132 doubles: the 8 lanes of a quarter-warp
// (g in 2 values x kq in 4) hit 8 distinct 16-byte bank groups.
constexpr int kGdPStride = 2 * 64 + 4;   // doubles per pair-row
constexpr int kGdPairRows = 32;          // 64 samples = 32 pair-rows
constexpr int kGdBlocksPerWarp = 3;   // 36 lower blocks of a 64x64 S over 12 warps
constexpr int kGdSlots = 3;           // raw tile ring (bulk copies in flight)
constexpr int kGdDBufs = DLX_GDA_DBUFS;   // centred operand tiles
constexpr size_t kGdRawBytes = static_cast<size_t>(kGdTile) * 64 * 8;
constexpr size_t kGdDBytes = static_cast<size_t>(kGdPairRows) * kGdPStride * 8;
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

// kFused = false: pass 2 proper, centring on the class means mu0 / mu1 (skipped entirely when
// *skip is set: the single-pass fit below already produced a certified S).
// kFused = true: the single-pass fit.  Centring is on a shift c_y (the class means of the
// first <= 64 rows, identical in every CTA), and the centring warps also accumulate the
// shifted class sums sum_{y_i = c}(x_i - c_c) and n1, so one read of x yields
// S' = sum (x - c_y)(x - c_y)^T, mu_c = c_c + sd_c / n_c and S = S' - sum_c sd_c sd_c^T / n_c.
template <bool kFused>
__global__ void __launch_bounds__(kGdThreads, 1)
gda_pass2_dmma_kernel(const double* __restrict__ x, const long long* __restrict__ y, int64_t n,
                      int d, const double* __restrict__ mu0, const double* __restrict__ mu1,
                      double* __restrict__ parts, const int* __restrict__ skip,
                      double* __restrict__ parts_sd, long long* __restrict__ parts_n1,
                      double* __restrict__ shift_out) {
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
  if (!kFused && skip != nullptr && *skip) return;   // uniform over the grid
  if (!kFused) {
    for (int j = tid; j < 128; j += kGdThreads) {
      const int c = j >> 6, jj = j & 63;
      mu_s[j] = jj < d ? (c ? mu1[jj] : mu0[jj]) : 0.0;
    }
  }
  __syncthreads();

  if (warp >= kGdMmaWarps) {
    // ---- centring warps: raw slot -> D[b] = x - mu_y (or x - c_y), zero outside n / d ------
    // thread = column pair (2cp, 2cp+1) x row phase rp: fixed columns, so the centre values
    // and the fused class sums live in registers
    const int ct = tid - kIssuer;
    const int cp = ct & 31, rp = ct >> 5, j0 = 2 * cp;
    if (ct == 0)
      for (int m = 0; m < kGdSlots && m < mt; ++m) issue(m);
    if (kFused) {
      // shift c_c = mean of the class-c rows among the first R <= 64 rows (all rows' mean for
      // a class absent there, 0 for n = 0); every CTA computes it in the same order
      const int R = static_cast<int>(std::min<int64_t>(n, 64));
      double2 q0 = make_double2(0.0, 0.0), q1 = q0;
      int k1 = 0;
      for (int r = rp; r < R; r += kGdCtrWarps) {
        const double vx = j0 < d ? x[static_cast<int64_t>(r) * d + j0] : 0.0;
        const double vy = j0 + 1 < d ? x[static_cast<int64_t>(r) * d + j0 + 1] : 0.0;
        const bool one = y[r] == 1;
        if (one) { q1.x += vx; q1.y += vy; ++k1; } else { q0.x += vx; q0.y += vy; }
      }
      double* red = Dbuf;   // free until the first tile is centred
      int* kred = reinterpret_cast<int*>(Dbuf + kGdCtrWarps * 128);
      *reinterpret_cast<double2*>(red + rp * 128 + j0) = q0;
      *reinterpret_cast<double2*>(red + rp * 128 + 64 + j0) = q1;
      if (cp == 0) kred[rp] = k1;
      named_bar(1, kGdCtrThreads);
      const int c = (ct >> 6) & 1, j = ct & 63;   // threads 0..127: (class, column)
      double sh = 0.0;
      if (ct < 128) {
        double t = 0.0, ta = 0.0;
        int kc = 0;
        for (int w = 0; w < kGdCtrWarps; ++w) {
          t += red[w * 128 + c * 64 + j];
          ta += red[w * 128 + j] + red[w * 128 + 64 + j];
          kc += kred[w];
        }
        const int k_c = c ? kc : R - kc;
        sh = k_c > 0 ? t / k_c : (R > 0 ? ta / R : 0.0);
      }
      named_bar(1, kGdCtrThreads);   // every read of red done before D is reused
      if (ct < 128) {
        mu_s[c * 64 + j] = j < d ? sh : 0.0;
        if (blockIdx.x == 0) shift_out[c * 64 + j] = j < d ? sh : 0.0;
        if (blockIdx.x == 0 && ct == 0) reinterpret_cast<unsigned*>(shift_out + 128)[0] = 0u;   // combine counter
      }
      named_bar(1, kGdCtrThreads);
    }
    // main loop mapping: lane = columns (ja, jb) = (cp, cp + 32), warp rp = pair-rows rp + 12 u
    const int ja = cp, jb = cp + 32;
    const double m0a = mu_s[ja], m0b = mu_s[jb], m1a = mu_s[64 + ja], m1b = mu_s[64 + jb];
    double a0a = 0.0, a0b = 0.0, a1a = 0.0, a1b = 0.0;   // fused: shifted class sums of my columns
    long long c1 = 0;                                    // fused: class-1 rows (cp == 0 threads)
    for (int m = 0; m < mt; ++m) {
      const int s = m % kGdSlots, b = m % kGdDBufs;
      const int64_t i0 = tile_of(m) * kGdTile;
      const int rows = static_cast<int>(std::min<int64_t>(kGdTile, n - i0));
      const bool from_smem = full_tile(m);
      mbar_wait(&raw_full[s], (m / kGdSlots) & 1);
      if (m >= kGdDBufs) mbar_wait(&d_empty[b], ((m - kGdDBufs) / kGdDBufs) & 1);
      const double* rs = raw + static_cast<size_t>(s) * kGdTile * 64;
      const long long* yv = ys + s * kGdTile;
      double* D = Dbuf + static_cast<size_t>(b) * kGdPairRows * kGdPStride;
      if (from_smem && d == 64) {
        // fast path: conflict-free 8-byte loads of two rows, 16-byte stores of (row, row + 4)
#pragma unroll 3
        for (int pr = rp; pr < kGdPairRows; pr += kGdCtrWarps) {
          const int r0 = (pr >> 2) * 8 + (pr & 3), r1 = r0 + 4;
          const double xa0 = rs[r0 * 64 + ja], xa1 = rs[r1 * 64 + ja];
          const double xb0 = rs[r0 * 64 + jb], xb1 = rs[r1 * 64 + jb];
          const bool one0 = yv[r0] == 1, one1 = yv[r1] == 1;
          double2 oa, ob;
          oa.x = xa0 - (one0 ? m1a : m0a);
          oa.y = xa1 - (one1 ? m1a : m0a);
          ob.x = xb0 - (one0 ? m1b : m0b);
          ob.y = xb1 - (one1 ? m1b : m0b);
          *reinterpret_cast<double2*>(D + pr * kGdPStride + 2 * ja) = oa;
          *reinterpret_cast<double2*>(D + pr * kGdPStride + 2 * jb) = ob;
          if (kFused) {
            // the label is warp-uniform (one row per warp): branch, so each element costs one
            // fp64 add for its class sum instead of two selects-and-adds
            if (one0) { a1a += oa.x; a1b += ob.x; } else { a0a += oa.x; a0b += ob.x; }
            if (one1) { a1a += oa.y; a1b += ob.y; } else { a0a += oa.y; a0b += ob.y; }
            c1 += one0 + one1;
          }
        }
      } else {
        for (int pr = rp; pr < kGdPairRows; pr += kGdCtrWarps) {
          const int r0 = (pr >> 2) * 8 + (pr & 3);
          double va[2] = {0.0, 0.0}, vb[2] = {0.0, 0.0};
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = r0 + 4 * h;
            if (r < rows) {
              const int64_t gi = i0 + r;
              const long long lab = from_smem ? yv[r] : __ldg(y + gi);
              const bool one = lab == 1;
              if (ja < d) va[h] = (from_smem ? rs[r * d + ja] : __ldg(x + gi * d + ja)) - (one ? m1a : m0a);
              if (jb < d) vb[h] = (from_smem ? rs[r * d + jb] : __ldg(x + gi * d + jb)) - (one ? m1b : m0b);
              if (kFused) {
                a1a += one ? va[h] : 0.0; a1b += one ? vb[h] : 0.0;
                a0a += one ? 0.0 : va[h]; a0b += one ? 0.0 : vb[h];
                c1 += one;
              }
            }
          }
          *reinterpret_cast<double2*>(D + pr * kGdPStride + 2 * ja) = make_double2(va[0], va[1]);
          *reinterpret_cast<double2*>(D + pr * kGdPStride + 2 * jb) = make_double2(vb[0], vb[1]);
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
    if (kFused) {
      // per-CTA partial record: sd_c[j] (ascending row-phase fold) and n1; raw slot 0 is free
      // (every tile has been consumed and no copy is outstanding)
      double* red = raw;
      long long* kred = reinterpret_cast<long long*>(raw + kGdCtrWarps * 128);
      red[rp * 128 + ja] = a0a;
      red[rp * 128 + jb] = a0b;
      red[rp * 128 + 64 + ja] = a1a;
      red[rp * 128 + 64 + jb] = a1b;
      if (cp == 0) kred[rp] = c1;
      named_bar(1, kGdCtrThreads);
      if (ct < 128) {
        const int c = ct >> 6, j = ct & 63;
        double t = 0.0;
        for (int w = 0; w < kGdCtrWarps; ++w) t += red[w * 128 + c * 64 + j];
        if (j < d) parts_sd[static_cast<size_t>(blockIdx.x) * 2 * d + c * d + j] = t;
      }
      if (ct == 0) {
        long long k = 0;
        for (int w = 0; w < kGdCtrWarps; ++w) k += kred[w];
        parts_n1[blockIdx.x] = k;
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
    const double* D = Dbuf + static_cast<size_t>(b) * kGdPairRows * kGdPStride;
    if (shared) {
#pragma unroll 2
      for (int k0 = 0; k0 < kGdTile; k0 += 8) {
        // one 16-byte load per index: .x = row k0 + kq, .y = row k0 + 4 + kq (column 8 idx + g)
        const double* prow = D + ((k0 >> 3) * 4 + kq) * kGdPStride + 2 * g;
        const double2 fa = *reinterpret_cast<const double2*>(prow + 16 * ba[0]);
#pragma unroll
        for (int u = 0; u < kGdBlocksPerWarp; ++u) {
          const double2 fb = *reinterpret_cast<const double2*>(prow + 16 * bb[u]);
          dmma_8x8x4(acc[u][0], fa.x, fb.x);
          dmma_8x8x4(acc[u][1], fa.y, fb.y);
        }
      }
    } else {
#pragma unroll 2
      for (int k0 = 0; k0 < kGdTile; k0 += 8) {
        const double* prow = D + ((k0 >> 3) * 4 + kq) * kGdPStride + 2 * g;
#pragma unroll
        for (int u = 0; u < kGdBlocksPerWarp; ++u)
          if (own[u]) {
            const double2 fa = *reinterpret_cast<const double2*>(prow + 16 * ba[u]);
            const double2 fb = *reinterpret_cast<const double2*>(prow + 16 * bb[u]);
            dmma_8x8x4(acc[u][0], fa.x, fb.x);
            dmma_8x8x4(acc[u][1], fa.y, fb.y);
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

// ---- d = 64: the k-split fit (r215-r218) ---------------------------------------------------
// The kernel above gives each tensor-core warp 3 of the 36 lower 8x8 blocks, so every warp
// reloads and every centring warp re-stores the whole tile (4 LDS.128 per 6 DMMAs).  Here the
// split is over samples instead: eight tensor-core warps (two per SM sub-partition, so one
// warp's loads and centring overlap the other's DMMAs) each own ALL 36 lower blocks (72 fp64
// accumulators per lane, 36 independent DMMA chains) for 8 of every 64-sample tile's rows, so
// a k-step costs 4 LDS.128 of x for 36 DMMAs; the warps centre their fragments in registers
// straight from the raw tile (no centred copy in shared memory) and, in the single-pass fit,
// also accumulate the shifted per-class sums from those centred fragments (one select-and-add
// per class), so no other warp touches the fp64 pipe the DMMAs use.
// One producer warp refills the 5-slot ring.
//
// Tiles arrive by TMA tensor copies (cp.async.bulk.tensor.2d, 4 boxes of 64 rows x 16 columns
// with the 128-byte swizzle: 16-byte chunk ch of row r sits at chunk ch ^ (r & 7) of the row's
// 128-byte line; rows past n are zero-filled by the TMA).  Lane (g, kq) loads, in box p, the
// chunk q(g) = (g >> 1) | ((g & 1) << 2) of sample row kq — i.e. physical columns
// 16p + 2q(g) + {0, 1} — and uses them as the LOGICAL columns 8(2p) + g and 8(2p+1) + g, so the
// accumulated S is S_phys under the column permutation P(8 idx + g) = 16 (idx >> 1) + 2 q(g) +
// (idx & 1), undone when the blocks are written.  With the swizzle, a quarter-warp's four rows
// x two chunks land in eight distinct 16-byte bank groups (no conflicts).  The eight warps'
// partial S and class sums are folded in ascending warp order through shared memory.
constexpr int kG64MmaWarps = 8;
constexpr int kG64Threads = (kG64MmaWarps + 4) * 32;   // + a warpgroup: the producer and 3 idle warps
// registers: 168 at launch; the tensor-core warpgroups take 240, the other drops to 24
constexpr int kG64RegsMma = 240, kG64RegsAux = 24;
static_assert(kG64MmaWarps * 32 * kG64RegsMma + 4 * 32 * kG64RegsAux <= 65536, "register budget");
#ifndef DLX_G64_ROWS
#define DLX_G64_ROWS 128
#endif
constexpr int kG64Rows = DLX_G64_ROWS;                  // samples per tile (8 or 16 rows per warp)
constexpr int kG64Steps = kG64Rows / (4 * kG64MmaWarps);   // k-steps per warp per tile
#ifndef DLX_G64_SLOTS
#define DLX_G64_SLOTS (kG64Rows == 64 ? 5 : 3)
#endif
constexpr int kG64Slots = DLX_G64_SLOTS;
constexpr size_t kG64BoxBytes = kG64Rows * 128;                            // kG64Rows rows x 16 doubles
constexpr size_t kG64RawBytes = 4 * kG64BoxBytes;
constexpr size_t kG64OffY = kG64Slots * kG64RawBytes;
constexpr size_t kG64OffMu = kG64OffY + kG64Slots * kG64Rows * 8;
constexpr int kG64Mu1 = 66;   // class-1 centre row: 16 bytes past a bank-aligned row, so lanes
                               // reading class-0 and class-1 centres of one column never collide
constexpr size_t kG64OffRed = kG64OffMu + 136 * 8;                        // shift fold
constexpr size_t kG64OffBar = kG64OffRed + kG64MmaWarps * 128 * 8 + 128;
constexpr size_t kG64Smem = kG64OffBar + 2 * kG64Slots * 8 + 1024;       // + base alignment slack
constexpr uint32_t kG64TxBytes = static_cast<uint32_t>(kG64RawBytes + kG64Rows * 8);
static_assert(kG64MmaWarps * (36 * 32 * 2 + 2 * 64) * 8 <= kG64OffY, "S fold must fit in the raw ring");

__host__ __device__ __forceinline__ int g64_q(int g) { return (g >> 1) | ((g & 1) << 2); }
__device__ __forceinline__ int g64_phys(int logical) {   // logical column 8 idx + g -> physical
  const int idx = logical >> 3, g = logical & 7;
  return 16 * (idx >> 1) + 2 * g64_q(g) + (idx & 1);
}

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_addr(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const CUtensorMap* map, int c0, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];" ::"r"(
          smem_addr(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(smem_addr(bar))
      : "memory");
}

template <bool kFused>
__global__ void __launch_bounds__(kG64Threads, 1)
gda_fit64_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmy,
                 const double* __restrict__ x, const long long* __restrict__ y, int64_t n,
                 const double* __restrict__ mu0, const double* __restrict__ mu1,
                 double* __restrict__ parts, const int* __restrict__ skip,
                 double* __restrict__ parts_sd, long long* __restrict__ parts_n1,
                 double* __restrict__ shift_out, double* __restrict__ S_out, unsigned* __restrict__ counter) {
  // S_out (pass 2 on given means, !kFused): the last CTA to finish folds the CTAs' records into
  // S_out itself (ascending CTA order) — the fit's fallback then needs no combine launch
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // the 128-byte swizzle needs 1024-byte aligned boxes; offsetting the shared array itself (not
  // an integer-cast address) keeps every access below an LDS rather than a generic load
  unsigned char* const smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  unsigned char* const raw = smem;
  long long* const ys = reinterpret_cast<long long*>(smem + kG64OffY);
  double* const mu_s = reinterpret_cast<double*>(smem + kG64OffMu);   // [mu0: 0..63 | mu1: 66..129]
  double* const red = reinterpret_cast<double*>(smem + kG64OffRed);
  uint64_t* const full = reinterpret_cast<uint64_t*>(smem + kG64OffBar);
  uint64_t* const empty = full + kG64Slots;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t ntiles = (n + kG64Rows - 1) / kG64Rows;
  const int mt = static_cast<int>(ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0);
  auto tile_of = [&](int m) { return static_cast<int64_t>(blockIdx.x) + static_cast<int64_t>(m) * gridDim.x; };
  auto rows_of = [&](int m) { return static_cast<int>(std::min<int64_t>(kG64Rows, n - tile_of(m) * kG64Rows)); };
  auto issue = [&](int m) {   // tile m -> slot m % kG64Slots (4 swizzled boxes + the labels)
    const int s = m % kG64Slots;
    const int row0 = static_cast<int>(tile_of(m) * kG64Rows);
    mbar_arrive_expect_tx(&full[s], kG64TxBytes);
#pragma unroll
    for (int p = 0; p < 4; ++p) tma_load_2d(raw + s * kG64RawBytes + p * kG64BoxBytes, &tmx, 16 * p, row0, &full[s]);
    tma_load_1d(ys + s * kG64Rows, &tmy, row0, &full[s]);
  };
  if (tid == 0) {
    for (int s = 0; s < kG64Slots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kG64MmaWarps);
    }
    fence_mbar_init();
  }
  pdl_wait();   // x / y / the means may come from the predecessor kernel
  pdl_trigger();
  if (!kFused && skip != nullptr && *skip) return;   // uniform over the grid
  if (!kFused)
    for (int j = tid; j < 128; j += kG64Threads) mu_s[j < 64 ? j : kG64Mu1 + j - 64] = j < 64 ? mu0[j] : mu1[j - 64];
  __syncthreads();

  if (warp >= kG64MmaWarps) {
    // ---- producer warp: keeps the ring kG64Slots tiles ahead of the slowest reader -----------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kG64RegsAux));
    if (warp == kG64MmaWarps && lane == 0) {
      for (int m = 0; m < mt; ++m) {
        if (m >= kG64Slots) {
          mbar_wait(&empty[m % kG64Slots], ((m - kG64Slots) / kG64Slots) & 1);
          fence_proxy_async_smem();
        }
        issue(m);
      }
    }
    __syncwarp();
    named_bar_split(3, kG64Threads);   // (A), met by the tensor-core warps below
    return;
  }

  if (kFused) {
    // shift c_c = mean of the class-c rows among the first R <= 64 rows (all R rows' mean for a
    // class absent there, 0 for n = 0); every CTA computes it in the same order.  Thread t:
    // column pair t & 31 (t & 31, + 32), rows (t >> 5) + 8u.
    const int R = static_cast<int>(std::min<int64_t>(n, 64));
    const int cp = tid & 31, rp = tid >> 5;
    double q0a = 0.0, q0b = 0.0, q1a = 0.0, q1b = 0.0;
    int k1 = 0;
    for (int r = rp; r < R; r += kG64MmaWarps) {
      const double va = x[static_cast<int64_t>(r) * 64 + cp], vb = x[static_cast<int64_t>(r) * 64 + cp + 32];
      if (y[r] == 1) { q1a += va; q1b += vb; ++k1; } else { q0a += va; q0b += vb; }
    }
    red[rp * 128 + cp] = q0a;
    red[rp * 128 + cp + 32] = q0b;
    red[rp * 128 + 64 + cp] = q1a;
    red[rp * 128 + 64 + cp + 32] = q1b;
    int* kred = reinterpret_cast<int*>(red + kG64MmaWarps * 128);
    if (cp == 0) kred[rp] = k1;
    named_bar(1, kG64MmaWarps * 32);
    double sh = 0.0;
    const int c = tid >> 6 & 1, j = tid & 63;   // threads 0..127: (class, column)
    if (tid < 128) {
      double t = 0.0, ta = 0.0;
      int kc = 0;
      for (int w = 0; w < kG64MmaWarps; ++w) {
        t += red[w * 128 + c * 64 + j];
        ta += red[w * 128 + j] + red[w * 128 + 64 + j];
        kc += kred[w];
      }
      const int k_c = c ? kc : R - kc;
      sh = k_c > 0 ? t / k_c : (R > 0 ? ta / R : 0.0);
    }
    named_bar(1, kG64MmaWarps * 32);   // every read of red done
    if (tid < 128) {
      mu_s[c * kG64Mu1 + j] = sh;
      if (blockIdx.x == 0) shift_out[c * 64 + j] = sh;
      if (blockIdx.x == 0 && tid == 0) reinterpret_cast<unsigned*>(shift_out + 128)[0] = 0u;   // combine counter
    }
    named_bar(1, kG64MmaWarps * 32);
  }

  // ---- tensor-core warps: rows 8 warp + 4 st + kq of every tile, all 36 lower blocks --------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kG64RegsMma));
  const int g = lane >> 2, kq = lane & 3, qg = g64_q(g);
  const double* mrow = mu_s + 2 * qg;   // + 64 c + 16 p: the centre pair of this lane's columns
  double acc[36][2];
#pragma unroll
  for (int b = 0; b < 36; ++b) acc[b][0] = acc[b][1] = 0.0;
  double sa[8], s1[8];   // fused: shifted sums of this lane's logical columns (class 0, class 1)
#pragma unroll
  for (int idx = 0; idx < 8; ++idx) sa[idx] = s1[idx] = 0.0;
  int c1 = 0;
  for (int m = 0; m < mt; ++m) {
    const int s = m % kG64Slots, rows = rows_of(m);
    mbar_wait(&full[s], (m / kG64Slots) & 1);
    const unsigned char* rs = raw + s * kG64RawBytes;
    const long long* yv = ys + s * kG64Rows;
#pragma unroll
    for (int st = 0; st < kG64Steps; ++st) {
      const int r = 4 * kG64Steps * warp + 4 * st + kq;
      const bool valid = r < rows;   // rows past n: zero-filled by the TMA, excluded here
      const bool one = yv[r] == 1;
      const unsigned char* rowp = rs + r * 128 + ((qg ^ (r & 7)) << 4);
      const double* mc = mrow + (one ? kG64Mu1 : 0);
      double f[8];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const double2 v = *reinterpret_cast<const double2*>(rowp + p * kG64BoxBytes);
        const double2 mu = *reinterpret_cast<const double2*>(mc + 16 * p);
        f[2 * p] = valid ? v.x - mu.x : 0.0;
        f[2 * p + 1] = valid ? v.y - mu.y : 0.0;
      }
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b <= a; ++b) dmma_8x8x4(acc[a * (a + 1) / 2 + b], f[a], f[b]);
      if (kFused) {
#pragma unroll
        // (selecting the class accumulator instead, one add per element, measured slower: r225)
        for (int idx = 0; idx < 8; ++idx) {   // per-class sums (all - class 1 would turn an
          sa[idx] += one ? 0.0 : f[idx];        // inf of class 1 into NaN for class 0)
          s1[idx] += one ? f[idx] : 0.0;
        }
        c1 += (valid && one) ? 1 : 0;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  named_bar_split(3, kG64Threads);   // (A) every tile consumed, no copy outstanding: the ring becomes the fold area
  double* fold = reinterpret_cast<double*>(raw);
#pragma unroll
  for (int b = 0; b < 36; ++b)
    *reinterpret_cast<double2*>(fold + ((warp * 36 + b) * 32 + lane) * 2) = make_double2(acc[b][0], acc[b][1]);
  double* fsum = fold + kG64MmaWarps * 36 * 64;   // [warp][class][logical column]
  if (kFused) {
    // class sums: fold the 4 row lanes (kq) of each column in order, then one lane per column
#pragma unroll
    for (int idx = 0; idx < 8; ++idx) {
      double va = sa[idx], v1 = s1[idx];
      va += __shfl_xor_sync(0xffffffffu, va, 1);
      v1 += __shfl_xor_sync(0xffffffffu, v1, 1);
      va += __shfl_xor_sync(0xffffffffu, va, 2);
      v1 += __shfl_xor_sync(0xffffffffu, v1, 2);
      if (kq == 0) {
        fsum[(warp * 2 + 0) * 64 + 8 * idx + g] = va;   // class 0
        fsum[(warp * 2 + 1) * 64 + 8 * idx + g] = v1;
      }
    }
    int k = c1;   // every lane of a row counts it: the g == 0 lanes hold one count per row
    k = g == 0 ? k : 0;
    for (int o = 16; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
    if (lane == 0) reinterpret_cast<long long*>(red)[warp] = k;
  }
  named_bar(2, kG64MmaWarps * 32);
  double* out = parts + static_cast<size_t>(blockIdx.x) * 4096;
  for (int e = tid; e < 36 * 32; e += kG64MmaWarps * 32) {
    const int b = e >> 5, ln = e & 31;
    double2 v = *reinterpret_cast<const double2*>(fold + (b * 32 + ln) * 2);
#pragma unroll
    for (int w = 1; w < kG64MmaWarps; ++w) {
      const double2 u = *reinterpret_cast<const double2*>(fold + ((w * 36 + b) * 32 + ln) * 2);
      v.x += u.x;
      v.y += u.y;
    }
    int a = 0;
    while ((a + 1) * (a + 2) / 2 <= b) ++a;
    const int bb = b - a * (a + 1) / 2;
    const int pr = g64_phys(8 * a + (ln >> 2));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int pc = g64_phys(8 * bb + 2 * (ln & 3) + h);
      const double val = h ? v.y : v.x;
      out[pr * 64 + pc] = val;
      if (a != bb) out[pc * 64 + pr] = val;
    }
  }
  if (kFused) {
    if (tid < 128) {   // (class, logical column) -> physical column, warps in ascending order
      const int c = tid >> 6, L = tid & 63;
      double t = 0.0;
      for (int w = 0; w < kG64MmaWarps; ++w) t += fsum[(w * 2 + c) * 64 + L];
      parts_sd[static_cast<size_t>(blockIdx.x) * 128 + c * 64 + g64_phys(L)] = t;
    }
    if (tid == 0) {
      long long k = 0;
      for (int w = 0; w < kG64MmaWarps; ++w) k += reinterpret_cast<const long long*>(red)[w];
      parts_n1[blockIdx.x] = k;
    }
  }
  if (!kFused && S_out != nullptr) {
    __shared__ int last;
    __threadfence();
    named_bar(2, kG64MmaWarps * 32);
    if (tid == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
    named_bar(2, kG64MmaWarps * 32);
    if (last) {
      __threadfence();
      for (int e = tid; e < 4096; e += kG64MmaWarps * 32) {
        double v = 0.0;
        for (unsigned p = 0; p < gridDim.x; ++p) v += __ldcg(parts + static_cast<size_t>(p) * 4096 + e);
        S_out[e] = v;
      }
      if (tid == 0) *counter = 0u;
    }
  }
}

// TMA tensor maps of x (n x 64 fp64, boxes of 64 rows x 16 columns, 128-byte swizzle) and y
// (n int64, boxes of 64), encoded per launch through the driver entry point (no libcuda link)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}
static int g64_maps(const double* x, const long long* y, int64_t n, CUtensorMap* tmx, CUtensorMap* tmy) {
  EncodeTiledFn enc = encode_tiled();
  DLX_REQUIRE(enc != nullptr, DLX_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t nn = static_cast<cuuint64_t>(std::max<int64_t>(n, 1));
  const cuuint64_t dx[2] = {64, nn}, sx[1] = {64 * 8};
  const cuuint32_t bx[2] = {16, static_cast<cuuint32_t>(kG64Rows)}, ex[2] = {1, 1};
  CUresult r = enc(tmx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(x), dx, sx, bx, ex,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DLX_REQUIRE(r == CUDA_SUCCESS, DLX_ERR_CUDA, "cuTensorMapEncodeTiled(x) failed");
  const cuuint64_t dy[1] = {nn}, sy[1] = {8};
  const cuuint32_t by[1] = {static_cast<cuuint32_t>(kG64Rows)}, ey[1] = {1};
  r = enc(tmy, CU_TENSOR_MAP_DATA_TYPE_INT64, 1, const_cast<long long*>(y), dy, sy, by, ey,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  DLX_REQUIRE(r == CUDA_SUCCESS, DLX_ERR_CUDA, "cuTensorMapEncodeTiled(y) failed");
  return DLX_OK;
}

// the k-split d = 64 kernel takes the bulk-copy ring: 16-byte aligned x and y
static bool gda_fit64_ok(const double* x, const long long* y, int d) {
  return d == 64 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0;
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
  if (gda_fit64_ok(x, y, d) && n > 0) {
    CUtensorMap tmx, tmy;
    if (int rc = g64_maps(x, y, n, &tmx, &tmy)) return rc;
    DLX_CUDA(cudaFuncSetAttribute(gda_fit64_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kG64Smem)));
    DLX_CUDA(launch_pdl(gda_fit64_kernel<false>, dim3(grid), dim3(kG64Threads), kG64Smem, stream, tmx, tmy, x, y, n, mu0,
                        mu1, parts, static_cast<const int*>(nullptr), static_cast<double*>(nullptr),
                        static_cast<long long*>(nullptr), static_cast<double*>(nullptr), static_cast<double*>(nullptr),
                        static_cast<unsigned*>(nullptr)));
    DLX_LAUNCHED("gda_fit64_kernel");
    return combine_f64(parts, grid, static_cast<long long>(d) * d, out, stream);
  }
  DLX_CUDA(cudaFuncSetAttribute(gda_pass2_dmma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kGdSmem)));
  DLX_CUDA(launch_pdl(gda_pass2_dmma_kernel<false>, dim3(grid), dim3(kGdThreads), kGdSmem, stream, x, y, n,
                      d, mu0, mu1, parts, static_cast<const int*>(nullptr), static_cast<double*>(nullptr),
                      static_cast<long long*>(nullptr), static_cast<double*>(nullptr)));
  DLX_LAUNCHED("gda_pass2_dmma_kernel");
  return combine_f64(parts, grid, static_cast<long long>(d) * d, out, stream);
}

// ---- the d = 64 single-pass fit on the int8 tensor cores (gda_fit_i8_kernel) ------------------
// S' = sum_i f_i f_i^T with f = fl(x - c_y) (the shift-centred rows, as the DMMA kernel forms them)
// computed as an EXACT integer product: every CTA quantises f per column to the fixed point
// Z_j = rne(f_j * 2^s_j) (s_j from the CTA's first tile: max |f_j| * 2^s_j < 2^42) and splits Z
// into six balanced base-256 digits e_0..e_5 (each in [-128, 127]; the bytes of Z + B, B = sum_i
// 128 * 2^(8i), with their top bit flipped — one FMA against a magic constant); with digit
// significance t = 5 - i, the digit products F_a^T F_b with t_a + t_b <= 5 (the dropped ones are
// below 2^-36 of the leading term) are four tcgen05 kind::i8 MMAs per 32-row step over digit
// pair groups G0 = {e5, e4}, G1 = {e3, e2}, G2 = {e1, e0}: (G0,G0), (G0,G1), (G0,G2), (G1,G1),
// each M = 128 (two digits x 64 columns) x N = 128, int32 accumulators resident in all 512 TMEM
// columns for the whole launch (a product <= 2^14 per row: exact for <= 2^17 rows per CTA).
// The off-diagonal group products enter S' with their transposes.  The class sums stay fp64
// sums of the same f (the means need them exactly as the DMMA path forms them).  Certification
// (gda_fit_combine): every CTA's quantum 2^-s_j must be <= 2^-30 of column j's RMS deviation,
// and a value outside the CTA's range (Z + B outside [0, 2^48), inf, NaN) sets the quantum to inf —
// either way *ok = 0 and the exact DMMA pass 2 on the means runs instead.
// 12 converter warps + the issuer + the producer: at most 4 warps per SM sub-partition, 128
// registers each.  The producer bulk-copies x / y tiles (96 contiguous rows = 48 KB) into two
// shared-memory stages, so the loads in flight do not cost converter registers.
constexpr int kI8Conv = 12;                           // converter warps (then the epilogue)
constexpr int kI8Threads = (kI8Conv + 2) * 32;        // + the MMA issuer and the producer warp
constexpr int kI8Rows = 96;                           // rows per tile: 4 passes of 24 (3 K-steps)
constexpr int kI8Stages = 2;                          // digit-plane buffers in flight
constexpr int kI8XStages = 3;                         // x / y tiles in flight
constexpr uint32_t kI8Group = kI8Rows * 128;          // one digit-pair group: 96 rows x 128 B
constexpr uint32_t kI8Stage = 3 * kI8Group;           // three groups per tile
constexpr uint32_t kI8XBytes = kI8Rows * 512;         // one x tile
constexpr size_t kI8OffX = kI8Stages * kI8Stage;
constexpr size_t kI8OffY = kI8OffX + kI8XStages * kI8XBytes;
constexpr size_t kI8OffMu = kI8OffY + kI8XStages * kI8Rows * 8;   // [c0: 0..63 | c1: 64..127] shift
constexpr size_t kI8OffScale = kI8OffMu + 128 * 8;    // 2^s_j
constexpr size_t kI8OffBar = kI8OffScale + 128 * 8;
constexpr size_t kI8Smem = kI8OffBar + (2 * kI8Stages + 2 * kI8XStages + 2) * 8 + 16 + 1024;
constexpr int kI8MaxTiles = (1 << 17) / kI8Rows;      // 2^17 rows per CTA (int32 exactness)
static_assert(2 * 128 * 129 * 4 <= kI8OffY, "TMEM staging must fit below the y stages");
static_assert(2 * kI8Conv * 128 * 8 <= kI8XStages * kI8XBytes, "class-sum fold fits in the x stages");
static_assert(kI8Smem <= 232448, "shared memory");
// plane byte L (the logical column) holds physical column i8_phys(L): converter c packs columns
// 2c, 2c+1, 32+2c, 33+2c, so a phase of 8 lanes reads 128 contiguous bytes of x (no conflicts)
__host__ __device__ constexpr int i8_phys(int L) { return (L & 3) < 2 ? 2 * (L >> 2) + (L & 3) : 32 + 2 * (L >> 2) + (L & 3) - 2; }

__global__ void __launch_bounds__(kI8Threads, 1)
gda_fit_i8_kernel(const double* __restrict__ x, const long long* __restrict__ y, int64_t n,
                  double* __restrict__ parts, double* __restrict__ parts_sd, long long* __restrict__ parts_n1,
                  double* __restrict__ parts_q, double* __restrict__ shift_out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* const smem = smem_raw + ((1024u - (smem_addr(smem_raw) & 1023u)) & 1023u);
  double* const mu_s = reinterpret_cast<double*>(smem + kI8OffMu);
  double* const sc_s = reinterpret_cast<double*>(smem + kI8OffScale);   // 2^s_j
  uint64_t* const pfull = reinterpret_cast<uint64_t*>(smem + kI8OffBar);
  uint64_t* const pempty = pfull + kI8Stages;
  uint64_t* const xfull = pempty + kI8Stages;
  uint64_t* const xempty = xfull + kI8XStages;
  uint64_t* const done = xempty + kI8XStages;
  uint32_t* const tmem_slot = reinterpret_cast<uint32_t*>(done + 2);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t ntiles = (n + kI8Rows - 1) / kI8Rows;
  const int mt = static_cast<int>(ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0);
  auto tile_row0 = [&](int m) { return (static_cast<int64_t>(blockIdx.x) + static_cast<int64_t>(m) * gridDim.x) * kI8Rows; };
  auto tile_rows = [&](int m) { return static_cast<int>(std::min<int64_t>(kI8Rows, n - tile_row0(m))); };
  if (tid == 0) {
    for (int s = 0; s < kI8Stages; ++s) {
      mbar_init(&pfull[s], kI8Conv);
      mbar_init(&pempty[s], 1);
    }
    for (int s = 0; s < kI8XStages; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], kI8Conv);
    }
    mbar_init(done, 1);
    fence_mbar_init();
    tmem_slot[1] = 0;   // range flag
  }
  if (warp == kI8Conv) tmem_alloc<512>(tmem_slot);
  pdl_wait();   // x / y may come from the predecessor kernel
  pdl_trigger();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kI8Conv) {
    // ---- MMA issuer: four group products per 32-row step, converged warp, lane 0 issues ----
    constexpr uint32_t ID = idesc_i8_major(128, 128, 1, 1, 1, 1);
    for (int m = 0; m < mt; ++m) {
      const int s = m % kI8Stages;
      mbar_wait(&pfull[s], (m / kI8Stages) & 1);
      tc_fence_after();
      const uint32_t b0 = smem_addr(smem + s * kI8Stage);
      if (lane == 0) {
#pragma unroll
        for (int kk = 0; kk < kI8Rows / 32; ++kk) {
          const uint64_t g0 = sw128_kmajor_desc(b0 + kk * 4096);
          const uint64_t g1 = sw128_kmajor_desc(b0 + kI8Group + kk * 4096);
          const uint64_t g2 = sw128_kmajor_desc(b0 + 2 * kI8Group + kk * 4096);
          const uint32_t acc = (m > 0 || kk > 0) ? 1u : 0u;
          mma_i8(tmem + 0, g0, g0, ID, acc);
          mma_i8(tmem + 128, g0, g1, ID, acc);
          mma_i8(tmem + 256, g0, g2, ID, acc);
          mma_i8(tmem + 384, g1, g1, ID, acc);
        }
        mma_commit(&pempty[s]);
      }
      __syncwarp();
    }
    if (lane == 0) mma_commit(done);
    __syncwarp();
  } else if (warp == kI8Conv + 1) {
    // ---- producer: x tile (contiguous rows) and the even part of its labels per stage; an odd
    // last label is read by its converter (bulk copies move multiples of 16 bytes) ----
    if (lane == 0) {
      for (int m = 0; m < mt; ++m) {
        const int xs = m % kI8XStages;
        if (m >= kI8XStages) mbar_wait(&xempty[xs], ((m - kI8XStages) / kI8XStages) & 1);
        const int64_t row0 = tile_row0(m);
        const uint32_t rows = static_cast<uint32_t>(tile_rows(m)), yb = (rows * 8u) & ~15u;
        mbar_arrive_expect_tx(&xfull[xs], rows * 512u + yb);
        bulk_g2s(smem + kI8OffX + xs * kI8XBytes, x + row0 * 64, rows * 512u, &xfull[xs]);
        if (yb) bulk_g2s(smem + kI8OffY + xs * kI8Rows * 8, y + row0, yb, &xfull[xs]);
      }
    }
    __syncwarp();
  } else {
    double* const red = reinterpret_cast<double*>(smem);   // prologue folds: the plane buffers
    // ---- converters: warp w, lane l: plane bytes 4c..4c+3 (c = l & 15; physical columns 2c,
    // 2c+1, 32+2c, 33+2c, i8_phys) of rows {r, r + 4} of an 8-row swizzle atom (disjoint bank
    // halves), 4 row passes of 24 rows per tile ----
    const int c = lane & 15, hsel = lane >> 4;
    const int rbase = (warp >> 2) * 8 + (warp & 3) + 4 * hsel;   // + 24 pass
    // shift c_y: class means of the first R <= 64 rows (every CTA, same order)
    {
      const int R = static_cast<int>(std::min<int64_t>(n, 64));
      const int cp = tid & 31, rp = tid >> 5;
      double q0a = 0.0, q0b = 0.0, q1a = 0.0, q1b = 0.0;
      int k1 = 0;
      for (int r = rp; r < R; r += kI8Conv) {
        const double va = x[static_cast<int64_t>(r) * 64 + cp], vb = x[static_cast<int64_t>(r) * 64 + cp + 32];
        if (y[r] == 1) { q1a += va; q1b += vb; ++k1; } else { q0a += va; q0b += vb; }
      }
      red[rp * 128 + cp] = q0a;
      red[rp * 128 + cp + 32] = q0b;
      red[rp * 128 + 64 + cp] = q1a;
      red[rp * 128 + 64 + cp + 32] = q1b;
      int* kred = reinterpret_cast<int*>(red + kI8Conv * 128);
      if (cp == 0) kred[rp] = k1;
      named_bar(1, kI8Conv * 32);
      if (tid < 128) {
        const int cl = tid >> 6, j = tid & 63;
        double t = 0.0, ta = 0.0;
        int kc = 0;
        for (int w = 0; w < kI8Conv; ++w) {
          t += red[w * 128 + cl * 64 + j];
          ta += red[w * 128 + j] + red[w * 128 + 64 + j];
          kc += kred[w];
        }
        const int k_c = cl ? kc : R - kc;
        const double sh = k_c > 0 ? t / k_c : (R > 0 ? ta / R : 0.0);
        mu_s[cl * 64 + j] = sh;
        if (blockIdx.x == 0) shift_out[cl * 64 + j] = sh;
        if (blockIdx.x == 0 && tid == 0) reinterpret_cast<unsigned*>(shift_out + 128)[0] = 0u;   // combine counter
      }
      named_bar(1, kI8Conv * 32);
    }
    // x / y of tile m, pass p: this thread's 4 columns of row 24 p + rbase (rows past the tile's
    // end read stale stage bytes and are excluded by their index)
    auto xrow = [&](int m, int p) {
      const double* xt = reinterpret_cast<const double*>(smem + kI8OffX + (m % kI8XStages) * kI8XBytes);
      const double* src = xt + (24 * p + rbase) * 64 + 2 * c;   // physical columns 2c, 2c+1 | 32+2c, 33+2c
      const double2 a = *reinterpret_cast<const double2*>(src), b = *reinterpret_cast<const double2*>(src + 32);
      return make_double4(a.x, a.y, b.x, b.y);
    };
    auto yrow = [&](int m, int p, int rows) {
      const int r = 24 * p + rbase;
      const long long* yt = reinterpret_cast<const long long*>(smem + kI8OffY + (m % kI8XStages) * kI8Rows * 8);
      if (r < (rows & ~1)) return yt[r];
      return r < rows ? __ldg(y + tile_row0(m) + r) : 0ll;
    };
    if (mt > 0) mbar_wait(&xfull[0], 0);
    // per-CTA scales from the first tile: max |f_j| over its rows
    {
      double mx[4] = {0.0, 0.0, 0.0, 0.0};
      const int rows0 = mt > 0 ? tile_rows(0) : 0;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        if (24 * p + rbase >= rows0) continue;
        const double4 v = xrow(0, p);
        const double* cc = mu_s + (yrow(0, p, rows0) == 1 ? 64 : 0);
        mx[0] = fmax(mx[0], fabs(v.x - cc[i8_phys(4 * c)]));
        mx[1] = fmax(mx[1], fabs(v.y - cc[i8_phys(4 * c + 1)]));
        mx[2] = fmax(mx[2], fabs(v.z - cc[i8_phys(4 * c + 2)]));
        mx[3] = fmax(mx[3], fabs(v.w - cc[i8_phys(4 * c + 3)]));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        mx[u] = fmax(mx[u], __shfl_xor_sync(0xffffffffu, mx[u], 16));
        if (hsel == 0) red[warp * 64 + i8_phys(4 * c + u)] = mx[u];
      }
      named_bar(1, kI8Conv * 32);
      if (tid < 64) {
        double m = 0.0;
        for (int w = 0; w < kI8Conv; ++w) m = fmax(m, red[w * 64 + tid]);   // NaN-free max (fmax)
        int s = 1000;   // an all-zero column: any nonzero value later is out of range
        if (m > 0.0 && m <= 1.0e300) s = 41 - ilogb(m);
        s = max(-1000, min(1000, s));
        sc_s[tid] = ldexp(1.0, s);
      }
      named_bar(1, kI8Conv * 32);
    }
    // the per-column scales in registers
    double scl[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) scl[u] = sc_s[i8_phys(4 * c + u)];
    bool bad = false;
    double sa[4] = {0.0, 0.0, 0.0, 0.0}, s1[4] = {0.0, 0.0, 0.0, 0.0};   // all rows, class 1
    int c1 = 0;
    constexpr double kMagic = 6755399441055744.0 + 141289400074368.0;   // 1.5 * 2^52 + B, B = 0x808080808080
    for (int m = 0; m < mt; ++m) {
      const int s = m % kI8Stages, rows = tile_rows(m);
      mbar_wait(&xfull[m % kI8XStages], (m / kI8XStages) & 1);
      if (m >= kI8Stages) mbar_wait(&pempty[s], ((m - kI8Stages) / kI8Stages) & 1);
      unsigned char* const gb = smem + s * kI8Stage;
      const long long* const yt = reinterpret_cast<const long long*>(smem + kI8OffY + (m % kI8XStages) * kI8Rows * 8);
      struct Row {   // one pass's operands: the row's 4 values, its class and its shift
        double4 xq;
        double2 ca, cb;
        bool one;
      };
      auto fetch = [&](auto full_tag, int p) {
        constexpr bool kFull = decltype(full_tag)::value;
        Row o;
        o.one = (kFull ? yt[24 * p + rbase] : yrow(m, p, rows)) == 1;
        o.xq = xrow(m, p);
        const double* cp = mu_s + (o.one ? 64 : 0) + 2 * c;   // the row's shift, same columns
        o.ca = *reinterpret_cast<const double2*>(cp);
        o.cb = *reinterpret_cast<const double2*>(cp + 32);
        return o;
      };
      auto do_pass = [&](auto full_tag, int p, const Row& o) {
        constexpr bool kFull = decltype(full_tag)::value;   // a whole tile: no row checks
        const int r = 24 * p + rbase;
        const bool valid = kFull || r < rows;
        const bool one = o.one;
        const double xv[4] = {o.xq.x, o.xq.y, o.xq.z, o.xq.w}, cc[4] = {o.ca.x, o.ca.y, o.cb.x, o.cb.y};
        // Z + B with B = sum_i 128 * 2^(8i) has plain bytes u_i (no carries): e_i = u_i - 128, i.e.
        // the byte u_i with its top bit flipped.  One FMA puts Z + B in the low 48 bits.
        uint32_t lo[4], hi[4];
        double f[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          f[u] = xv[u] - cc[u];
          if (!kFull) f[u] = valid ? f[u] : 0.0;   // padding rows: zero digits, no class
          const long long bits = __double_as_longlong(fma(f[u], scl[u], kMagic));
          lo[u] = static_cast<uint32_t>(bits);
          hi[u] = static_cast<uint32_t>(bits >> 32);
        }
        // class sums without selects: all rows (a padding row adds f = 0) and class 1 through an
        // FMA with the row's 0 / 1 weight, on the fp64 pipe; class 0 = all - class 1.  Only a
        // non-finite value (inf * 0 = NaN) breaks that — it also sets the range flag, and the
        // CTA then recomputes its class sums directly (below)
        const double w1 = one ? 1.0 : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          sa[u] += f[u];
          s1[u] = fma(f[u], w1, s1[u]);
        }
        // in range iff 0 <= Z + B < 2^48, i.e. the top 16 bits are the magic's (also false for
        // inf / NaN and for |f 2^s| >= 2^51)
        constexpr uint32_t K = 0x43380000u;
        bad |= ((((hi[0] ^ K) | (hi[1] ^ K)) | ((hi[2] ^ K) | (hi[3] ^ K))) >> 16) != 0u;
        // 4 x 6 byte transpose: word i holds digit i of the 4 columns (column u in byte u)
        const uint32_t t01l = __byte_perm(lo[0], lo[1], 0x5140), t01h = __byte_perm(lo[0], lo[1], 0x7362);
        const uint32_t t23l = __byte_perm(lo[2], lo[3], 0x5140), t23h = __byte_perm(lo[2], lo[3], 0x7362);
        const uint32_t h01 = __byte_perm(hi[0], hi[1], 0x5140), h23 = __byte_perm(hi[2], hi[3], 0x5140);
        uint32_t w[6];
        w[0] = __byte_perm(t01l, t23l, 0x5410) ^ 0x80808080u;
        w[1] = __byte_perm(t01l, t23l, 0x7632) ^ 0x80808080u;
        w[2] = __byte_perm(t01h, t23h, 0x5410) ^ 0x80808080u;
        w[3] = __byte_perm(t01h, t23h, 0x7632) ^ 0x80808080u;
        w[4] = __byte_perm(h01, h23, 0x5410) ^ 0x80808080u;
        w[5] = __byte_perm(h01, h23, 0x7632) ^ 0x80808080u;
        c1 += (valid && one) ? 1 : 0;
        // group g holds (e_{5-2g} at bytes 0..63, e_{4-2g} at bytes 64..127)
        // (asm stores without a memory clobber: the compiler may hoist the next pass's shared
        // loads above them — the planes are only read by the tensor cores, after the fence below)
        const uint32_t gs = smem_addr(gb);
#pragma unroll
        for (int g = 0; g < 3; ++g) {
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(gs + g * kI8Group + sw128_offset(r, 4 * c)), "r"(w[5 - 2 * g]));
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(gs + g * kI8Group + sw128_offset(r, 64 + 4 * c)), "r"(w[4 - 2 * g]));
        }
      };
      if (rows == kI8Rows) {
        Row cur = fetch(std::true_type{}, 0);
#pragma unroll
        for (int p = 0; p < 4; ++p) {   // the next pass's shared loads issue before this pass's math
          Row nxt = cur;
          if (p < 3) nxt = fetch(std::true_type{}, p + 1);
          do_pass(std::true_type{}, p, cur);
          cur = nxt;
        }
      } else {
#pragma unroll
        for (int p = 0; p < 4; ++p) do_pass(std::false_type{}, p, fetch(std::false_type{}, p));
      }
      fence_proxy_async_smem();   // generic-proxy stores -> visible to the tensor cores
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&pfull[s]);
        mbar_arrive(&xempty[m % kI8XStages]);
      }
    }
    // ---- class sums, counts, range flag: fixed-order folds through shared memory ----
    int* const flag_s = reinterpret_cast<int*>(tmem_slot + 1);
    if (bad) atomicOr(flag_s, 1);
    double* const rede = reinterpret_cast<double*>(smem + kI8OffX);   // every x stage consumed
    named_bar(1, kI8Conv * 32);
    if (*flag_s == 0) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        rede[(warp * 2 + hsel) * 128 + i8_phys(4 * c + u)] = sa[u] - s1[u];   // class 0
        rede[(warp * 2 + hsel) * 128 + 64 + i8_phys(4 * c + u)] = s1[u];
      }
    } else {
      // a value outside the CTA's range (possibly inf / NaN): the exact per-class sums of the
      // CTA's rows, re-read from global memory (thread: column tid & 63, rows of group tid >> 6)
      constexpr int kG = kI8Conv * 32 / 64;
      const int j = tid & 63, rg = tid >> 6;
      double q0 = 0.0, q1 = 0.0;
      for (int m = 0; m < mt; ++m) {
        const int64_t row0 = tile_row0(m);
        const int rows = tile_rows(m);
        for (int r = rg; r < rows; r += kG) {
          const double f = x[(row0 + r) * 64 + j] - mu_s[(y[row0 + r] == 1 ? 64 : 0) + j];
          if (y[row0 + r] == 1) q1 += f; else q0 += f;
        }
      }
      for (int q = tid; q < 2 * kI8Conv * 128; q += kI8Conv * 32) rede[q] = 0.0;
      named_bar(1, kI8Conv * 32);
      rede[rg * 128 + j] = q0;
      rede[rg * 128 + 64 + j] = q1;
    }
    int k1 = c == 0 ? c1 : 0;   // each row is counted by its 16 column lanes: keep one
    for (int o = 16; o > 0; o >>= 1) k1 += __shfl_xor_sync(0xffffffffu, k1, o);
    int* const kred = reinterpret_cast<int*>(sc_s + 64);   // the upper half of the scale area
    named_bar(1, kI8Conv * 32);
    if (lane == 0) kred[warp] = k1;
    if (tid < 128) {
      double t = 0.0;
      for (int q = 0; q < 2 * kI8Conv; ++q) t += rede[q * 128 + tid];
      parts_sd[static_cast<size_t>(blockIdx.x) * 128 + tid] = t;
    }
    named_bar(1, kI8Conv * 32);
    if (tid == 0) {
      long long kk = 0;
      for (int w = 0; w < kI8Conv; ++w) kk += kred[w];
      parts_n1[blockIdx.x] = kk;
    }
    if (tid < 64)   // the CTA's quantum per column; inf when a value fell outside its range
      parts_q[static_cast<size_t>(blockIdx.x) * 64 + tid] =
          *flag_s ? __longlong_as_double(0x7ff0000000000000ll) : 1.0 / sc_s[tid];
    // ---- S' from the four group products: TMEM -> padded staging -> fixed-order cell sums ----
    mbar_wait(done, 0);
    tc_fence_after();
    if (mt == 0) {   // no tile: the accumulators were never written
      for (int e = tid; e < 4096; e += kI8Conv * 32) parts[static_cast<size_t>(blockIdx.x) * 4096 + e] = 0.0;
    } else {
    int* const stage = reinterpret_cast<int*>(smem);   // [2][128][129] int32 (the plane buffers)
    const int qd = warp & 3, cc = warp >> 2;   // lane quarter (warp rank in its warpgroup), chunk
    constexpr int kJ = kI8Conv * 32 / 64;      // rows j per pass: cells (j0 + kJ v, k)
    constexpr int kV = (64 + kJ - 1) / kJ;
    double acc[kV];
#pragma unroll
    for (int v = 0; v < kV; ++v) acc[v] = 0.0;
    const int k = tid & 63, j0 = tid >> 6;
#pragma unroll 1
    for (int R = 0; R < 2; ++R) {
      for (int ch = cc; ch < 4; ch += kI8Conv / 4) {   // 64-column chunks of this round
        const int gi = ch >> 1, n0 = (ch & 1) * 64;
        int* const row = stage + (gi * 128 + 32 * qd + lane) * 129 + n0;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          int32_t v[16];
          tmem_ld16(tmem + (static_cast<uint32_t>(32 * qd) << 16) + R * 256 + ch * 64 + 16 * h, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) row[16 * h + i] = v[i];
        }
      }
      named_bar(1, kI8Conv * 32);
#pragma unroll
      for (int gi = 0; gi < 2; ++gi) {
        const int P = 2 * R + gi;
        const int pp = P == 3 ? 1 : 0, qq = P == 3 ? 1 : P;   // (0,0) (0,1) (0,2) (1,1)
        const int* const D = stage + gi * 128 * 129;
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const double wgt = ldexp(1.0, 8 * ((5 - (2 * pp + a)) + (5 - (2 * qq + b))));
#pragma unroll
            for (int v = 0; v < kV; ++v) {
              const int j = min(j0 + kJ * v, 63);
              acc[v] += wgt * static_cast<double>(D[(a * 64 + j) * 129 + b * 64 + k]);
              if (pp != qq) acc[v] += wgt * static_cast<double>(D[(a * 64 + k) * 129 + b * 64 + j]);
            }
          }
      }
      named_bar(1, kI8Conv * 32);
    }
    // S' symmetric by construction: (j, k) and (k, j) both take the value formed for the cell
    // with j <= k (the two are sums of the same products in different orders)
    double* const sym = reinterpret_cast<double*>(smem);   // [64][65], the staging is consumed
#pragma unroll
    for (int v = 0; v < kV; ++v) {
      const int j = j0 + kJ * v;
      if (j < 64 && j <= k) sym[j * 65 + k] = acc[v];
    }
    named_bar(1, kI8Conv * 32);
    double* const out = parts + static_cast<size_t>(blockIdx.x) * 4096;
    const int pk = i8_phys(k), sk = ilogb(sc_s[pk]);
#pragma unroll
    for (int v = 0; v < kV; ++v) {
      const int j = j0 + kJ * v;
      if (j < 64) {
        const int pj = i8_phys(j);
        out[pj * 64 + pk] = scalbn(sym[min(j, k) * 65 + max(j, k)], -(ilogb(sc_s[pj]) + sk));
      }
    }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kI8Conv) tmem_dealloc<512>(tmem);
}

// Single-pass fit, last step (gda_fit_combine, combine.cu): mu_c = c_c + sd_c / n_c and
// S = S' - sum_c sd_c sd_c^T / n_c.  Certified: the rank-1 corrections may cancel at most 99 % of
// any diagonal entry of S' (relative rounding amplification <= 100); otherwise *ok = 0 and the
// caller's pass 2 on the exact means runs (gda_pass2_dmma_kernel<false> / combine gated on *ok).

size_t gda_fit_workspace_bytes(int64_t n, int d) {
  const int grid = gda_pass2_dmma_grid(n);
  Carve c(nullptr);
  c.take<double>(static_cast<size_t>(grid) * d * d);
  c.take<double>(static_cast<size_t>(grid) * 2 * d);
  c.take<long long>(grid);
  c.take<double>(static_cast<size_t>(d) * d);
  c.take<double>(2 * static_cast<size_t>(d));
  c.take<long long>(1);
  c.take<double>(129);
  c.take<int>(1);
  c.take<double>(static_cast<size_t>(grid) * 64);   // int8 fit: the CTAs' quanta
  c.take<double>(64);
  return c.used + 256;
}

int gda_fit_combine(const double* parts, const double* parts_sd, const long long* parts_n1, int nparts, int d,
                    double* Sp, double* sd, long long* n1p, int64_t n, const double* shift, unsigned* counter,
                    long long* n1_out, double* mu0, double* mu1, double* S, int* ok, cudaStream_t s,
                    const double* parts_q = nullptr, double* qmax = nullptr);

// the int8 fit (DLX_GDA_I8=0 keeps the DMMA fit): d = 64, aligned rows, <= 2^17 rows per CTA
static bool gda_i8_enabled() {   // read per fit (tests switch it in-process)
  const char* e = std::getenv("DLX_GDA_I8");
  return e == nullptr || e[0] != '0';
}

// 2 = int8 fit, 1 = k-split DMMA fit, 0 = row blocks (dlx_gda_fit_path)
int gda_fit_path(const double* x, const long long* y, int64_t n, int d) {
  if (!(gda_fit64_ok(x, y, d) && n > 0 && !std::getenv("DLX_GDA_ROWBLOCKS"))) return 0;
  const int grid = gda_pass2_dmma_grid(n);
  const int64_t i8_tiles = (n + kI8Rows - 1) / kI8Rows;
  return gda_i8_enabled() && (i8_tiles + grid - 1) / grid <= kI8MaxTiles ? 2 : 1;
}

int gda_fit(const double* x, const long long* y, int64_t n, int d, long long* n1_out, double* mu0,
            double* mu1, double* S, void* ws, size_t ws_bytes, cudaStream_t stream) {
  DLX_REQUIRE(n >= 0 && d > 0, DLX_ERR_ARG, "gda fit: bad shape");
  DLX_REQUIRE(d <= 64, DLX_ERR_GENERATION, "GenerationFailed: single-pass GDA fit needs d <= 64");
  const int grid = gda_pass2_dmma_grid(n);
  Carve c(ws);
  double* parts = c.take<double>(static_cast<size_t>(grid) * d * d);
  double* parts_sd = c.take<double>(static_cast<size_t>(grid) * 2 * d);
  long long* parts_n1 = c.take<long long>(grid);
  double* Sp = c.take<double>(static_cast<size_t>(d) * d);
  double* sd = c.take<double>(2 * static_cast<size_t>(d));
  long long* n1 = c.take<long long>(1);
  double* shift = c.take<double>(129);   // + the combine's completion counter
  int* ok = c.take<int>(1);
  double* parts_q = c.take<double>(static_cast<size_t>(grid) * 64);
  double* qmax = c.take<double>(64);
  DLX_REQUIRE(ws && c.used <= ws_bytes, DLX_ERR_ARG, "gda fit: workspace too small");
  const int path = gda_fit_path(x, y, n, d);
  const bool k64 = path >= 1, i8 = path == 2;
  CUtensorMap tmx, tmy;
  if (i8) {
    if (int rc = g64_maps(x, y, n, &tmx, &tmy)) return rc;   // for the fallback pass
    DLX_CUDA(cudaFuncSetAttribute(gda_fit_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kI8Smem)));
    DLX_CUDA(cudaFuncSetAttribute(gda_fit64_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kG64Smem)));
    DLX_CUDA(launch_pdl(gda_fit_i8_kernel, dim3(grid), dim3(kI8Threads), kI8Smem, stream, x, y, n, parts,
                        parts_sd, parts_n1, parts_q, shift));
    DLX_LAUNCHED("gda_fit_i8_kernel");
  } else if (k64) {
    if (int rc = g64_maps(x, y, n, &tmx, &tmy)) return rc;
    DLX_CUDA(cudaFuncSetAttribute(gda_fit64_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kG64Smem)));
    DLX_CUDA(cudaFuncSetAttribute(gda_fit64_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kG64Smem)));
    DLX_CUDA(launch_pdl(gda_fit64_kernel<true>, dim3(grid), dim3(kG64Threads), kG64Smem, stream, tmx, tmy, x, y, n,
                        static_cast<const double*>(nullptr), static_cast<const double*>(nullptr), parts,
                        static_cast<const int*>(nullptr), parts_sd, parts_n1, shift, static_cast<double*>(nullptr),
                        static_cast<unsigned*>(nullptr)));
    DLX_LAUNCHED("gda_fit64_kernel");
  } else {
    DLX_CUDA(cudaFuncSetAttribute(gda_pass2_dmma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kGdSmem)));
    DLX_CUDA(cudaFuncSetAttribute(gda_pass2_dmma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kGdSmem)));
    DLX_CUDA(launch_pdl(gda_pass2_dmma_kernel<true>, dim3(grid), dim3(kGdThreads), kGdSmem, stream, x, y, n, d,
                        static_cast<const double*>(nullptr), static_cast<const double*>(nullptr), parts,
                        static_cast<const int*>(nullptr), parts_sd, parts_n1, shift));
    DLX_LAUNCHED("gda_pass2_dmma_kernel");
  }
  // combine + finalize in one launch (combine.cu); shift[128] is its completion counter, zeroed
  // by the fit kernel's block 0
  if (int rc = gda_fit_combine(parts, parts_sd, parts_n1, grid, d, Sp, sd, n1, n, shift,
                               reinterpret_cast<unsigned*>(shift + 128), n1_out, mu0, mu1, S, ok, stream,
                               i8 ? parts_q : nullptr, qmax))
    return rc;
  // fallback, decided on the device: pass 2 on the exact means when the shift was too far off
  if (k64) {   // folds its own records into S when it runs (no combine launch)
    DLX_CUDA(launch_pdl(gda_fit64_kernel<false>, dim3(grid), dim3(kG64Threads), kG64Smem, stream, tmx, tmy, x, y, n,
                        static_cast<const double*>(mu0), static_cast<const double*>(mu1), parts,
                        static_cast<const int*>(ok), static_cast<double*>(nullptr),
                        static_cast<long long*>(nullptr), static_cast<double*>(nullptr), S,
                        reinterpret_cast<unsigned*>(shift + 128)));
    DLX_LAUNCHED("gda_fit64_kernel");
    return DLX_OK;
  } else {
    DLX_CUDA(launch_pdl(gda_pass2_dmma_kernel<false>, dim3(grid), dim3(kGdThreads), kGdSmem, stream, x, y, n, d,
                        static_cast<const double*>(mu0), static_cast<const double*>(mu1), parts,
                        static_cast<const int*>(ok), static_cast<double*>(nullptr),
                        static_cast<long long*>(nullptr), static_cast<double*>(nullptr)));
    DLX_LAUNCHED("gda_pass2_dmma_kernel");
  }
  return combine_f64_unless(parts, grid, static_cast<long long>(d) * d, S, ok, stream);
}

// Sharded fit: rank r's single-pass fit gives n_rc, mu_rc and S_r (its scatter around its own
// class means).  With every rank's (n_rc, mu_rc) summed into a table (rank r fills row r, the
// other rows are zero, so the sum is exact) and the S_r summed, the global result follows from
// the pooled-scatter identity  S = sum_r S_r + sum_r sum_c n_rc (mu_rc - mu_c)(mu_rc - mu_c)^T,
// mu_c = sum_r n_rc mu_rc / n_c — the between-rank term computed directly from the differences
// (no cancellation), ranks folded in ascending order.  Ranks without class-c rows are skipped.
__global__ void __launch_bounds__(1024)
gda_combine_ranks_kernel(const double* __restrict__ table, int world, int d, double* __restrict__ S,
                         long long* __restrict__ n1_out, double* __restrict__ mu0, double* __restrict__ mu1) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ double mu_s[];   // [2][d] global class means
  const int w = 2 + 2 * d;
  double n[2] = {0.0, 0.0};
  for (int r = 0; r < world; ++r) {
    n[0] += table[r * w];
    n[1] += table[r * w + 1];
  }
  for (int e = threadIdx.x; e < 2 * d; e += blockDim.x) {
    const int c = e / d, j = e % d;
    double acc = 0.0;
    for (int r = 0; r < world; ++r) {
      const double nr = table[r * w + c];
      if (nr > 0.0) acc += nr * table[r * w + 2 + c * d + j];
    }
    const double m = acc / n[c];   // an empty class: 0 / 0 -> NaN, as the reference
    mu_s[e] = m;
    (c ? mu1 : mu0)[j] = m;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < d * d; e += blockDim.x) {
    const int a = e / d, b = e % d;
    double acc = S[e];
    for (int r = 0; r < world; ++r)
      for (int c = 0; c < 2; ++c) {
        const double nr = table[r * w + c];
        if (nr > 0.0) {
          const double* mr = table + r * w + 2 + c * d;
          acc += nr * ((mr[a] - mu_s[c * d + a]) * (mr[b] - mu_s[c * d + b]));
        }
      }
    S[e] = acc;
  }
  if (threadIdx.x == 0) *n1_out = static_cast<long long>(n[1]);
}

}  // namespace dlx

extern "C" {

int dlx_gda_combine_ranks(const double* d_table, int32_t world, int32_t d, double* d_scatter,
                          int64_t* d_n1, double* d_mu0, double* d_mu1, dlx_stream_t stream) {
  DLX_REQUIRE(d_table && d_scatter && d_n1 && d_mu0 && d_mu1 && world >= 1 && d > 0 && d <= 4096,
              DLX_ERR_ARG, "gda combine ranks: bad args");
  const size_t smem = 2 * static_cast<size_t>(d) * sizeof(double);
  DLX_CUDA(dlx::launch_pdl(dlx::gda_combine_ranks_kernel, dim3(1), dim3(1024), smem, static_cast<cudaStream_t>(stream),
                      d_table, static_cast<int>(world), static_cast<int>(d), d_scatter,
                      reinterpret_cast<long long*>(d_n1), d_mu0, d_mu1));
  DLX_LAUNCHED("gda_combine_ranks_kernel");
  return DLX_OK;
}


size_t dlx_gda_fit_workspace_bytes(int64_t n, int32_t d) { return dlx::gda_fit_workspace_bytes(n, d); }

int dlx_gda_fit(const double* d_x, const int64_t* d_y, int64_t n, int32_t d, int64_t* d_n1,
                double* d_mu0, double* d_mu1, double* d_scatter, void* d_workspace,
                size_t workspace_bytes, dlx_stream_t stream) {
  return dlx::gda_fit(d_x, reinterpret_cast<const long long*>(d_y), n, d, reinterpret_cast<long long*>(d_n1),
                      d_mu0, d_mu1, d_scatter, d_workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
}

int dlx_gda_fit_path(const void* d_x, const void* d_y, int64_t n, int32_t d, int* h_path) {
  DLX_REQUIRE(h_path && n >= 0 && d > 0, DLX_ERR_ARG, "gda fit path: bad args");
  *h_path = dlx::gda_fit_path(static_cast<const double*>(d_x), static_cast<const long long*>(d_y), n, d);
  return DLX_OK;
}

int dlx_gda_fit_last_fallback(const void* d_workspace, int64_t n, int32_t d, int* h_fallback) {
  // the certification flag of the last dlx_gda_fit on this workspace (synchronous read)
  DLX_REQUIRE(d_workspace && h_fallback, DLX_ERR_ARG, "gda fit: bad args");
  dlx::Carve c(const_cast<void*>(d_workspace));
  const int grid = dlx::gda_pass2_dmma_grid(n);
  c.take<double>(static_cast<size_t>(grid) * d * d);
  c.take<double>(static_cast<size_t>(grid) * 2 * d);
  c.take<long long>(grid);
  c.take<double>(static_cast<size_t>(d) * d);
  c.take<double>(2 * static_cast<size_t>(d));
  c.take<long long>(1);
  c.take<double>(129);
  int* ok = c.take<int>(1);
  int h = 0;
  DLX_CUDA(cudaMemcpy(&h, ok, sizeof(int), cudaMemcpyDeviceToHost));
  *h_fallback = !h;
  return DLX_OK;
}

}  // extern "C"
