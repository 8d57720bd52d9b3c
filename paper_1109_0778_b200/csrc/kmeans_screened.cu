// kmeans_screened.cu — the k-means fused multiloop with a tcgen05 int8 distance screen and an
// exact fp64 recheck.  Assignments stay bit-identical to the reference argmin chain
// (proj/src/stage.cpp:73-104 staged_if chain over the inner mk_reduce distances,
// loops.cpp:111-174), while the per-sample work drops from k*d fp64 (x-mu)^2 chains to one
// small integer GEMM tile plus, for the rare near-ties, a few exact chains.
//
// Why a screen: the direct form costs 3*N*k*d fp64 ops (2.1e11 per C4 iteration, ~11 ms at
// the FP64 pipe peak) against 1.34 ms of HBM time.  argmin_c (x-mu_c)^2 =
// argmin_c (|mu_c|^2 - 2 x.mu_c), and x.mu_c is a GEMM.  We compute it EXACTLY on integer
// tensor cores for 23-bit fixed-point copies of x and mu, bound the fixed-point error
// rigorously, and only re-evaluate the reference's own fp64 chain where the bound cannot
// separate the best centroid from the others.
//
// Fixed point.  Per tile e_t with |x| < 2^e_t; per launch e_m with |mu| < 2^e_m over finite
// centroids.  Y = rint(x * 2^(22-e_t)), |Y| <= 2^22, split Y = 65536 h + 256 l + F with h in
// s8 and l, F in u8 (same for mu: Y' = 65536 h' + 256 l' + G).  tcgen05.mma kind::i8 computes
// exact int32 accumulators
//   HH = sum h h',  CR = sum (h l' + l h'),  W1 = sum (h G + F h' + l l'),  W2 = sum (l G + F l')
// so sum Y Y' = 2^32 HH + 2^24 CR + 2^16 W1 + 2^8 W2 + sum F G  (the last term, in [0, d*255^2],
// is dropped).  With x~ = Y + phi, mu~ = Y' + gamma, |phi|,|gamma| <= 1/2:
//   sum x~ mu~ = sum Y Y' + E,  |E| <= (sum|Y| + sum|Y'|)/2 + d/4.
// In units U = 2^(e_t+e_m-20), x.mu/U = sum x~ mu~ / 2^24 and Q = 256 HH + CR + (W1>>8) +
// (W2>>16) satisfies x.mu/U in [Q - e, Q + 2.25 + e], e = ((sum|Y|+sum|Y'|)/2 + d/4)/2^24.
// The screened score T_c = floor(|mu_c|^2/U) - 2 Q_c brackets |mu_c|^2/U - 2 x.mu_c/U within
// [T_c - 4.5 - 2e, T_c + 1 + 2e], and the reference's fp64 chain differs from the real
// distance by < 1 unit (guarded by -8 <= e_m - e_t <= 2, |e| <= 400).  So every centroid with
//   T_c > min_c T_c + W,   W = 9 + ceil(4 e),   (sum|Y| <= d 2^22 per sample, sum|Y'| <= max_c)
// has a strictly larger reference distance than some other centroid and cannot be the argmin.
// One survivor => it IS the reference argmin.  Several survivors => the sample goes to the
// pending list and is re-evaluated with the reference chain (sequential j, no FMA, strict <,
// ascending c, start (1e300, 0)).  Tiles with non-finite values or out-of-range exponents
// send every sample to the exact chain.  NaN / inf centroids never win the reference chain
// and are excluded from the screen.
//
// Kernel shape: one persistent CTA per SM, 14 warps, warp-specialised around mbarriers:
//   warp 0      TMA producer: 1-D bulk copies of 112-sample x tiles into a 3-stage ring
//   warp 1      TMEM owner + MMA issuer (one thread): 16 tcgen05.mma per tile into a
//               double-buffered 4 x 64-column int32 accumulator
//   warps 2-5   converters: tile exponent, rint(x*2^(22-e)) via the fp64 magic-number add,
//               byte split into the SW128 [h|l] and SW64 [F] K-major A operands
//   warps 6-13  epilogue + bucket-reduce: tcgen05.ld the accumulators and screen; samples with
//               a unique survivor are stably counting-sorted by centroid and folded into
//               register-resident per-centroid sums (warp w owns centroids w, w+8, ...; lane
//               l owns columns 2l, 2l+1; rows folded in ascending order: deterministic, no
//               atomics); samples with several survivors (and every sample of a guarded
//               tile) go to a per-CTA pending list
//   resolve     a second small kernel evaluates the reference chain for the pending samples
//               (one thread per (sample, candidate) pair), writes their assignments and folds
//               their rows into per-CTA partial records, in list order (deterministic).
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "sm100.cuh"

namespace dlx {

int kmeans_finalize(const long long* part_counts, const double* part_sums, int parts, int k, int d,
                    long long* counts, double* sums, cudaStream_t stream);

namespace sk {

using namespace sm100;

constexpr int kThreads = 512;
constexpr int kTile = 112;        // samples per tile (the MMA runs M=128; rows 112..127 are zero)
constexpr int kMmaM = 128;
constexpr int kStages = 3;
constexpr int kMaxD = 64;
constexpr int kMaxK = 64;
// warp roles: 0 = TMA producer; 1 = TMEM owner + MMA issuer; 2-7 converters; 8-11 epilogue
// (TMEM lane quarters 0-3); 12-15 fold
constexpr int kWarpProd = 0, kWarpMma = 1, kWarpC0 = 2, kNumC = 6, kWarpE0 = 8, kWarpR0 = 12;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kAccCols = 256;                        // 4 accumulators x 64 columns
constexpr uint32_t kXStage = kTile * kMaxD * 8;           // 56 KiB
constexpr uint32_t kOffA1 = kStages * kXStage;            // [h|l]  128 x 128 B, SW128
constexpr uint32_t kOffA2 = kOffA1 + kMmaM * 128;         // [F]    128 x 64 B,  SW64
constexpr uint32_t kOffB1 = kOffA2 + kMmaM * 64;          // [h'|l'] 64 x 128 B, SW128
constexpr uint32_t kOffB2 = kOffB1 + kMaxK * 128;         // [G]     64 x 64 B,  SW64
constexpr uint32_t kOffMisc = kOffB2 + kMaxK * 64;
static_assert(kOffA1 % 1024 == 0 && kOffB1 % 1024 == 0 && kOffA2 % 512 == 0 && kOffB2 % 512 == 0,
              "UMMA operand alignment");
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52: x + kMagic rounds x to an integer

constexpr int kListCap = 16;  // fold list slots per owned centroid per tile

struct Misc {
  uint64_t full[kStages], sempty[kStages], cfull[kStages], efull[kStages];
  uint64_t a_full, a_empty, tfull[2], tempty[2];
  unsigned long long valid;
  uint32_t tmem_base;
  int em, yabs, disabled, window;
  uint32_t mu_maxhi;
  alignas(16) int nm0[kMaxK];             // floor(|mu_c|^2 / U), U = 2^(e_t + e_m - 20), e_t = e_m + 1
  double nmf[kMaxK];
  unsigned char rowflag[kStages][kMmaM];  // sample needs the exact chain (|x| >= 2^e_t, inf, NaN)
  int pcount[2][4];
  uint32_t gm[kStages][4][kMaxK];         // per stage, per quarter: rows of the tile resolved to c
  unsigned char list[4][16][kListCap];    // per fold warp, per owned centroid: rows, ascending
};
constexpr uint32_t kSmemBytes = kOffMisc + sizeof(Misc);
static_assert(kSmemBytes <= 232448, "shared-memory plan exceeds 227 KiB");
constexpr int kInvalidNm = 0x70000000;  // > any valid score (|Q| < 2^26, nm <= 2^25)
constexpr int kNoCandidate = 0x60000000;

__device__ __forceinline__ int exp_bound(uint32_t maxhi) {
  // smallest e with |v| < 2^e for the largest |v| whose high word (sans sign) is maxhi
  return static_cast<int>(maxhi >> 20) - 1022;
}

// byte offset of (row, byte k) inside a K-major SWIZZLE_64B operand with 64-byte rows
__device__ __forceinline__ uint32_t sw64_offset(uint32_t row, uint32_t kbyte) {
  const uint32_t chunk = (kbyte >> 4) ^ ((row & 7) >> 1);
  return (row >> 3) * 512u + (row & 7) * 64u + (chunk << 4) + (kbyte & 15);
}

// rint(v) for |v| < 2^31 as the low word of v + 1.5*2^52 (one fp64 add, exact scaling before)
__device__ __forceinline__ int rint_magic(double scaled) {
  return __double2loint(__dadd_rn(scaled, kMagic));
}
// rint(x * scale) for a power-of-two scale: the product is exact, so one fma rounds once
__device__ __forceinline__ int rint_fma(double x, double scale) {
  return __double2loint(__fma_rn(x, scale, kMagic));
}

__global__ void __launch_bounds__(kThreads, 1)
kmeans_screened_kernel(const double* __restrict__ x, int64_t n, int d, int k,
                       const double* __restrict__ mu, int32_t* __restrict__ assign,
                       long long* __restrict__ part_counts, double* __restrict__ part_sums,
                       long long* __restrict__ pend_idx, unsigned long long* __restrict__ pend_mask,
                       long long* __restrict__ pend_count, long long pend_cap,
                       long long* __restrict__ trace) {
  extern __shared__ __align__(1024) unsigned char smem[];
  Misc& S = *reinterpret_cast<Misc*>(smem + kOffMisc);
  // optional per-role cycle accounting (build with -DDLX_KMEANS_TRACE, run with
  // DLX_KMEANS_TRACE=1): lane 0 of one warp per role
#ifdef DLX_KMEANS_TRACE
  long long tr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long t0 = clock64();
#define TR(slot) do { const long long _t = clock64(); tr[slot] += _t - t0; t0 = _t; } while (0)
#else
#define TR(slot) do { } while (0)
#endif
  unsigned char* A1 = smem + kOffA1;
  unsigned char* A2 = smem + kOffA2;
  unsigned char* B1 = smem + kOffB1;
  unsigned char* B2 = smem + kOffB2;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (n + kTile - 1) / kTile;
  const int mtiles = static_cast<int>((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x);

  // ---- prologue: barriers, B operands (fixed-point centroids), per-centroid constants ------
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&S.full[s], 1);
      mbar_init(&S.sempty[s], 4);
      mbar_init(&S.cfull[s], kNumC);
      mbar_init(&S.efull[s], 4);
    }
    mbar_init(&S.a_full, kNumC);
    mbar_init(&S.a_empty, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&S.tfull[b], 1);
      mbar_init(&S.tempty[b], 4);
    }
    S.valid = 0;
    S.yabs = 0;
    S.mu_maxhi = 0;
    fence_mbar_init();
  }
  __syncthreads();
  if (tid < kMaxK) {  // per centroid: validity (all finite), max |mu| high word, |mu|^2
    const int c = tid;
    uint32_t mx = 0;
    bool ok = c < k;
    double nm = 0.0;
    if (ok) {
      for (int j = 0; j < d; ++j) {
        const double v = mu[c * d + j];
        const uint32_t hw = static_cast<uint32_t>(__double2hiint(v)) & 0x7fffffffu;
        if (hw >= 0x7ff00000u) ok = false;
        mx = max(mx, hw);
        nm += v * v;
      }
    }
    S.nmf[c] = nm;
    if (ok) {
      atomicOr(&S.valid, 1ull << c);
      atomicMax(&S.mu_maxhi, mx);
    }
  }
  __syncthreads();
  if (tid == 0) {
    const int em = S.mu_maxhi == 0 ? 0 : exp_bound(S.mu_maxhi);
    S.em = em;
    S.disabled = (em > 400 || em < -400) ? 1 : 0;
  }
  __syncthreads();
  {
    const double scale = S.disabled ? 0.0 : ldexp(1.0, 22 - S.em);
    const unsigned long long valid = S.valid;
    for (int e = tid; e < kMaxK * kMaxD; e += kThreads) {
      const int c = e / kMaxD, j = e - c * kMaxD;
      int Y = 0;
      if (((valid >> c) & 1) && j < d) Y = rint_magic(mu[c * d + j] * scale);
      B1[sw128_offset(c, j)] = static_cast<unsigned char>(Y >> 16);
      B1[sw128_offset(c, 64 + j)] = static_cast<unsigned char>(Y >> 8);
      B2[sw64_offset(c, j)] = static_cast<unsigned char>(Y);
    }
    if (tid < kMaxK && ((valid >> tid) & 1)) {
      int sa = 0;
      for (int j = 0; j < d; ++j) sa += abs(rint_magic(mu[tid * d + j] * scale));
      atomicMax(&S.yabs, sa);
    }
  }
  __syncthreads();
  if (tid < kMaxK) {  // per-launch score constants (the sample exponent is fixed at e_t = e_m + 1)
    const unsigned long long valid = S.valid;
    S.nm0[tid] = (S.disabled || !((valid >> tid) & 1))
                     ? kInvalidNm
                     : __double2int_rd(S.nmf[tid] * ldexp(1.0, 19 - 2 * S.em));
    if (tid == 0) {
      // W = 9 + ceil(4e), e = ((d*2^22 + max_c sum|Y'|)/2 + d/4) / 2^24  (+1 margin)
      const long long num = (static_cast<long long>(d) << 22) + S.yabs;
      S.window = 10 + static_cast<int>((2 * num + d + (1ll << 24) - 1) >> 24);
    }
  }
  fence_proxy_async_smem();
  if (warp == kWarpMma) tmem_alloc<kTmemCols>(&S.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;

  if (warp == kWarpProd) {
    // ======================= TMA producer =======================
    if (lane == 0) {
      for (int m = 0; m < mtiles; ++m) {
        const int64_t t = blockIdx.x + static_cast<int64_t>(m) * gridDim.x;
        const int s = m % kStages;
        TR(1);
        if (m >= kStages) mbar_wait(&S.sempty[s], ((m / kStages) - 1) & 1);
        TR(0);
        const int rows = static_cast<int>(n - t * kTile < kTile ? n - t * kTile : kTile);
        const uint32_t bytes = static_cast<uint32_t>(rows) * d * 8u;
        mbar_arrive_expect_tx(&S.full[s], bytes);
        bulk_g2s(smem + s * kXStage, x + t * kTile * d, bytes, &S.full[s]);
      }
    }
  } else if (warp == kWarpMma) {
    // ======================= MMA issuer =======================
    if (lane == 0) {
      // A pieces: h (s8), l (u8), F (u8); B pieces: h' (s8), l' (u8), G (u8)
      constexpr uint32_t ID_hh = idesc_i8(kMmaM, 64, 1, 1);
      constexpr uint32_t ID_hu = idesc_i8(kMmaM, 64, 1, 0);
      constexpr uint32_t ID_uh = idesc_i8(kMmaM, 64, 0, 1);
      constexpr uint32_t ID_uu = idesc_i8(kMmaM, 64, 0, 0);
      const uint32_t a1 = smem_addr(A1), a2 = smem_addr(A2), b1 = smem_addr(B1), b2 = smem_addr(B2);
      const int nk = (d + 31) / 32;
      for (int m = 0; m < mtiles; ++m) {
        const int b = m & 1;
        TR(2);
        mbar_wait(&S.a_full, m & 1);
        TR(0);
        if (m >= 2) mbar_wait(&S.tempty[b], ((m >> 1) - 1) & 1);
        TR(1);
        tc_fence_after();
        const uint32_t dt = tmem + b * kAccCols;
        for (int kk = 0; kk < nk; ++kk) {
          const uint64_t xh = sw128_kmajor_desc(a1 + 32 * kk), xl = sw128_kmajor_desc(a1 + 64 + 32 * kk);
          const uint64_t xf = sw64_kmajor_desc(a2 + 32 * kk);
          const uint64_t mh = sw128_kmajor_desc(b1 + 32 * kk), ml = sw128_kmajor_desc(b1 + 64 + 32 * kk);
          const uint64_t mg = sw64_kmajor_desc(b2 + 32 * kk);
          const uint32_t acc = kk > 0;
          mma_i8(dt + 0, xh, mh, ID_hh, acc);      // HH
          mma_i8(dt + 64, xh, ml, ID_hu, acc);     // CR = h l' + l h'
          mma_i8(dt + 64, xl, mh, ID_uh, 1);
          mma_i8(dt + 128, xh, mg, ID_hu, acc);    // W1 = h G + F h' + l l'
          mma_i8(dt + 128, xf, mh, ID_uh, 1);
          mma_i8(dt + 128, xl, ml, ID_uu, 1);
          mma_i8(dt + 192, xl, mg, ID_uu, acc);    // W2 = l G + F l'
          mma_i8(dt + 192, xf, ml, ID_uu, 1);
        }
        mma_commit(&S.a_empty);
        mma_commit(&S.tfull[b]);
      }
    }
  } else if (warp >= kWarpC0 && warp < kWarpC0 + kNumC) {
    // ======================= converters (6 warps) =======================
    const int cw = warp - kWarpC0;
    const int em = S.em, disabled = S.disabled;
    const double scale = disabled ? 0.0 : ldexp(1.0, 21 - em);   // 2^(22 - e_t), e_t = e_m + 1
    const uint32_t hw_limit = static_cast<uint32_t>(1023 + em + 1) << 20;  // |x| >= 2^e_t
    const int half = lane >> 4, j0 = 4 * (lane & 15);
    const bool colok = j0 < d, col2ok = j0 + 2 < d;
    for (int m = 0; m < mtiles; ++m) {
      const int64_t t = blockIdx.x + static_cast<int64_t>(m) * gridDim.x;
      const int s = m % kStages;
      const int rows = static_cast<int>(n - t * kTile < kTile ? n - t * kTile : kTile);
      TR(4);
      mbar_wait(&S.full[s], (m / kStages) & 1);
      TR(0);
      const double* xs = reinterpret_cast<const double*>(smem + s * kXStage);
      if (m >= 1) mbar_wait(&S.a_empty, (m - 1) & 1);
      TR(2);
      // Y = rint(x * 2^(22-e_t)) with e_t = e_m + 1 fixed per launch; row pairs (2p, 2p+1),
      // p = cw, cw + 6, ...; lane (half, lane16) converts columns 4*lane16 .. +3 of row 2p+half.
      // A row with |x| >= 2^e_t, inf or NaN is flagged (exact chain).
#pragma unroll 2
      for (int pp = cw; pp < kMmaM / 2; pp += kNumC) {
        const int q = 2 * pp + half;
        const bool ok = q < rows && colok;
        const double* src = ok ? xs + q * d + j0 : xs;
        const double2 v0 = *reinterpret_cast<const double2*>(src);
        const double2 v1 = (ok && col2ok) ? *reinterpret_cast<const double2*>(src + 2) : make_double2(0.0, 0.0);
        const double a0 = ok ? v0.x : 0.0, a1 = ok ? v0.y : 0.0;
        const uint32_t hx = max(max(static_cast<uint32_t>(__double2hiint(a0)) & 0x7fffffffu,
                                    static_cast<uint32_t>(__double2hiint(a1)) & 0x7fffffffu),
                                max(static_cast<uint32_t>(__double2hiint(v1.x)) & 0x7fffffffu,
                                    static_cast<uint32_t>(__double2hiint(v1.y)) & 0x7fffffffu));
        const unsigned badm = __ballot_sync(0xffffffffu, hx >= hw_limit);
        if ((lane & 15) == 0) S.rowflag[s][q] = static_cast<unsigned char>(
            disabled || ((badm >> (16 * half)) & 0xffffu) != 0);
        const int Y0 = rint_fma(a0, scale), Y1 = rint_fma(a1, scale);
        const int Y2 = rint_fma(v1.x, scale), Y3 = rint_fma(v1.y, scale);
        // bytes of Y (little endian): b0 = F, b1 = l, b2 = h (low byte of Y >> 16)
        const uint32_t p01 = __byte_perm(Y0, Y1, 0x6240), p23 = __byte_perm(Y2, Y3, 0x6240);
        const uint32_t q01 = __byte_perm(Y0, Y1, 0x0051), q23 = __byte_perm(Y2, Y3, 0x0051);
        const uint32_t oh = sw128_offset(q, j0);
        *reinterpret_cast<uint32_t*>(A1 + oh) = __byte_perm(p01, p23, 0x7632);                 // h
        *reinterpret_cast<uint32_t*>(A1 + (oh ^ 64u)) = __byte_perm(q01, q23, 0x5410);         // l
        *reinterpret_cast<uint32_t*>(A2 + sw64_offset(q, j0)) = __byte_perm(p01, p23, 0x5410);  // F
      }
      TR(3);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&S.a_full);
        mbar_arrive(&S.cfull[s]);
      }
    }
  } else if (warp >= kWarpE0 && warp < kWarpR0) {
    // ======================= epilogue: screen + decide (4 warps, one per lane quarter) ===========
    const int quarter = warp & 3;
    const int q = quarter * 32 + lane;  // sample row within the tile (M row)
    const unsigned long long kmask = k == 64 ? ~0ull : ((1ull << k) - 1);
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    const int window = S.window;
    long long* my_pidx = pend_idx + static_cast<size_t>(blockIdx.x) * pend_cap;
    unsigned long long* my_pmask = pend_mask + static_cast<size_t>(blockIdx.x) * pend_cap;
    long long pending = 0;
    const int4* nm4 = reinterpret_cast<const int4*>(S.nm0);
    for (int m = 0; m < mtiles; ++m) {
      const int64_t t = blockIdx.x + static_cast<int64_t>(m) * gridDim.x;
      const int s = m % kStages, b = m & 1;
      const int rows = static_cast<int>(n - t * kTile < kTile ? n - t * kTile : kTile);
      TR(6);
      mbar_wait(&S.cfull[s], (m / kStages) & 1);
      TR(0);
      mbar_wait(&S.tfull[b], (m >> 1) & 1);
      TR(1);
      tc_fence_after();
      int tv[64];
      int lmin = kInvalidNm;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        const uint32_t col = b * kAccCols + 8 * ch;
        int hh[8], cr[8], w1[8], w2[8];
        tmem_ld8(tmem + lane_base + col, hh);
        tmem_ld8(tmem + lane_base + col + 64, cr);
        tmem_ld8(tmem + lane_base + col + 128, w1);
        tmem_ld8(tmem + lane_base + col + 192, w2);
        const int4 n0 = nm4[2 * ch], n1 = nm4[2 * ch + 1];
        const int nm[8] = {n0.x, n0.y, n0.z, n0.w, n1.x, n1.y, n1.z, n1.w};
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          // invalid centroids: zero B rows (Q = 0) and nm = kInvalidNm
          const int Q = hh[u] * 256 + cr[u] + (w1[u] >> 8) + (w2[u] >> 16);
          const int v = nm[u] - 2 * Q;
          tv[8 * ch + u] = v;
          lmin = min(lmin, v);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.tempty[b]);
      TR(2);
      unsigned long long full = 0;
      bool pend = false;
      int a = -1;
      if (q < rows) {
        if (S.rowflag[s][q]) {
          full = kmask;  // |x| out of the screen's range, inf or NaN: the exact chain over all c
          pend = true;
        } else if (lmin < kNoCandidate) {
          const int thr = lmin + window;
#pragma unroll
          for (int u = 0; u < 64; ++u)
            if (tv[u] <= thr) full |= 1ull << u;
          if ((full & (full - 1)) == 0) {
            a = __ffsll(static_cast<long long>(full)) - 1;
          } else {
            pend = true;  // several survivors: resolved by the exact chain (resolve kernel)
          }
        } else {
          a = 0;  // no finite centroid: the chain keeps its start index
        }
        if (a >= 0 && assign) assign[t * kTile + q] = a;
      }
      // group masks for the fold: gm[s][quarter][c] = this quarter's rows resolved to c
      const unsigned grp = __match_any_sync(0xffffffffu, a);
      S.gm[s][quarter][lane] = 0u;
      S.gm[s][quarter][lane + 32] = 0u;
      __syncwarp();
      if ((grp & ((1u << lane) - 1)) == 0 && a >= 0) S.gm[s][quarter][a] = grp;
      // deterministic pending-list append, ordered by sample row
      const unsigned pb = __ballot_sync(0xffffffffu, pend);
      if (lane == 0) S.pcount[m & 1][quarter] = __popc(pb);
      named_bar(1, 128);
      const int p0 = S.pcount[m & 1][0], p1 = S.pcount[m & 1][1], p2 = S.pcount[m & 1][2];
      if (pend) {
        const int before = (quarter > 0 ? p0 : 0) + (quarter > 1 ? p1 : 0) + (quarter > 2 ? p2 : 0);
        const long long slot = pending + before + __popc(pb & ((1u << lane) - 1));
        my_pidx[slot] = t * kTile + q;
        my_pmask[slot] = full;
      }
      pending += p0 + p1 + p2 + S.pcount[m & 1][3];
      TR(3);
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.efull[s]);
    }
    if (quarter == 0 && lane == 0) pend_count[blockIdx.x] = pending;
  } else {
    // ======================= fold: bucket-reduce (4 warps) =======================
    // Warp rw owns centroids rw + 4u (u = 0..15); lane (u, g) = (lane >> 1, lane & 1) owns
    // columns 32g .. 32g+31 of centroid rw + 4u as 16 pairs visited in the rotated order
    // (i + u) % 16, so one LDS.128 of the warp spreads over all banks; acc[i] holds pair
    // (i + u) % 16.  Rows are folded in ascending order: deterministic, no atomics.
    const int rw = warp - kWarpR0;
    const int u = lane >> 1, g = lane & 1;
    const int c = rw + 4 * u;
    double acc[16][2];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = 0.0;
    long long cnt_lane = 0;  // rows of centroid c in quarters 2g, 2g+1
    for (int m = 0; m < mtiles; ++m) {
      const int s = m % kStages;
      TR(6);
      mbar_wait(&S.efull[s], (m / kStages) & 1);
      mbar_wait(&S.full[s], (m / kStages) & 1);
      TR(0);
      const double* xs = reinterpret_cast<const double*>(smem + s * kXStage);
      // row list of centroid c: quarters 0,1 (lane 2u) then 2,3 (lane 2u+1), lanes ascending
      const unsigned ma = S.gm[s][2 * g][c], mb = S.gm[s][2 * g + 1][c];
      const int pc = __popc(ma) + __popc(mb);
      cnt_lane += pc;
      const int up = __shfl_up_sync(0xffffffffu, pc, 1), dn = __shfl_down_sync(0xffffffffu, pc, 1);
      const int before = g ? up : 0;          // rows of quarters 0,1 precede quarters 2,3
      const int nu = g ? up + pc : pc + dn;   // rows of centroid c this tile
      int slot = before;
      unsigned mm = ma;
      while (mm) {
        const int l = __ffs(mm) - 1;
        mm &= mm - 1;
        if (slot < kListCap) S.list[rw][u][slot] = static_cast<unsigned char>(64 * g + l);
        ++slot;
      }
      mm = mb;
      while (mm) {
        const int l = __ffs(mm) - 1;
        mm &= mm - 1;
        if (slot < kListCap) S.list[rw][u][slot] = static_cast<unsigned char>(64 * g + 32 + l);
        ++slot;
      }
      const int rounds = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(nu)));
      __syncwarp();
      TR(1);
      const int lim = min(rounds, kListCap);
      for (int t4 = 0; t4 < lim; ++t4) {
        if (t4 < nu) {
          const double* xr = xs + S.list[rw][u][t4] * d + 32 * g;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int pr = (i + u) & 15;
            if (32 * g + 2 * pr < d) {
              const double2 w = *reinterpret_cast<const double2*>(xr + 2 * pr);
              acc[i][0] += w.x;
              acc[i][1] += w.y;
            }
          }
        }
      }
      if (rounds > kListCap) {  // crowded centroid: walk the quarter masks directly (same order)
        int seen = 0;
        for (int Qr = 0; Qr < 4; ++Qr) {
          unsigned gg = S.gm[s][Qr][c];
          while (gg) {
            const int row = 32 * Qr + __ffs(gg) - 1;
            gg &= gg - 1;
            if (seen++ < kListCap) continue;
            const double* xr = xs + row * d + 32 * g;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int pr = (i + u) & 15;
              if (32 * g + 2 * pr < d) {
                const double2 w = *reinterpret_cast<const double2*>(xr + 2 * pr);
                acc[i][0] += w.x;
                acc[i][1] += w.y;
              }
            }
          }
        }
      }
      TR(4);
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.sempty[s]);
    }
    // flush this CTA's partial activation record
    if (c < k) {
      double* ps = part_sums + static_cast<size_t>(blockIdx.x) * k * d + static_cast<size_t>(c) * d;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int col = 32 * g + 2 * ((i + u) & 15);
        if (col < d) ps[col] = acc[i][0];
        if (col + 1 < d) ps[col + 1] = acc[i][1];
      }
    }
    const long long ct = cnt_lane + __shfl_xor_sync(0xffffffffu, cnt_lane, 1);
    if (g == 0 && c < k) part_counts[static_cast<size_t>(blockIdx.x) * k + c] = ct;
  }
#ifdef DLX_KMEANS_TRACE
  if (trace && lane == 0 &&
      (warp == kWarpProd || warp == kWarpMma || warp == kWarpC0 || warp == kWarpE0 || warp == kWarpR0)) {
    const int role = warp == kWarpProd ? 0 : warp == kWarpMma ? 1 : warp == kWarpC0 ? 2 : warp == kWarpE0 ? 3 : 4;
    for (int i = 0; i < 8; ++i) trace[(static_cast<size_t>(blockIdx.x) * 5 + role) * 8 + i] = tr[i];
  }
#endif
#undef TR
  __syncthreads();
  if (warp == kWarpMma) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

// ---------------------------------------------------------------------------------------
// resolve: the reference chain for the pending samples.  Resolve CTA rb handles slice
// rb % kResSplit of main-kernel CTA rb / kResSplit's pending list, in chunks of kResChunk
// samples: the chunk's rows are gathered into shared memory next to the fp64 centroids,
// every (sample, candidate) pair is one thread's exact chain (sequential j, no FMA), each
// sample then merges its candidates in ascending centroid order (strict <, NaN never
// wins, start (1e300, 0)), and the rows are folded into this CTA's partial record in list
// order (deterministic).
constexpr int kResThreads = 256;
constexpr int kResSplit = 4;
constexpr int kResChunk = 64;
constexpr int kResMaxPairs = kResChunk * kMaxK;

__global__ void __launch_bounds__(kResThreads)
kmeans_resolve_kernel(const double* __restrict__ x, int d, int k, const double* __restrict__ mu,
                      int32_t* __restrict__ assign, const long long* __restrict__ pend_idx,
                      const unsigned long long* __restrict__ pend_mask,
                      const long long* __restrict__ pend_count, long long pend_cap,
                      long long* __restrict__ part_counts, double* __restrict__ part_sums) {
  extern __shared__ double rsm[];
  double* mu_s = rsm;                          // k*d
  double* sums_s = mu_s + k * d;               // k*d
  double* rows_s = sums_s + k * d;             // kResChunk*d
  double* dist_s = rows_s + kResChunk * d;     // kResMaxPairs
  __shared__ long long idx_s[kResChunk];
  __shared__ unsigned long long mask_s[kResChunk];
  __shared__ int first_s[kResChunk + 1];
  __shared__ int a_s[kResChunk];
  __shared__ long long cnt_s[kMaxK];
  const int tid = threadIdx.x;
  const int src = blockIdx.x / kResSplit, slice = blockIdx.x % kResSplit;
  const long long total = pend_count[src];
  const long long lo = total * slice / kResSplit, hi = total * (slice + 1) / kResSplit;
  const long long* pidx = pend_idx + static_cast<size_t>(src) * pend_cap;
  const unsigned long long* pmask = pend_mask + static_cast<size_t>(src) * pend_cap;
  for (int e = tid; e < k * d; e += kResThreads) {
    mu_s[e] = mu[e];
    sums_s[e] = 0.0;
  }
  for (int c = tid; c < k; c += kResThreads) cnt_s[c] = 0;
  constexpr int R = kResThreads / 64;
  const int jj = tid & 63, rr = tid >> 6;
  for (long long base = lo; base < hi; base += kResChunk) {
    const int nrow = static_cast<int>(hi - base < kResChunk ? hi - base : kResChunk);
    __syncthreads();
    for (int e = tid; e < nrow; e += kResThreads) {
      idx_s[e] = pidx[base + e];
      mask_s[e] = pmask[base + e];
    }
    __syncthreads();
    if (tid < 32) {  // exclusive scan of candidate counts -> pair offsets
      int run = 0;
      for (int e0 = 0; e0 < nrow; e0 += 32) {
        const int e = e0 + tid;
        const int c = e < nrow ? __popcll(mask_s[e]) : 0;
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, incl, o);
          if (tid >= o) incl += t;
        }
        if (e < nrow) first_s[e] = run + incl - c;
        run += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (tid == 0) first_s[nrow] = run;
    }
    for (int e = tid; e < nrow * d; e += kResThreads) {
      const int r = e / d, j = e - r * d;
      rows_s[e] = __ldg(x + idx_s[r] * d + j);
    }
    __syncthreads();
    const int npairs = first_s[nrow];
    for (int p = tid; p < npairs; p += kResThreads) {
      int r = 0;  // owning sample: last r with first_s[r] <= p
      for (int step = kResChunk; step > 0; step >>= 1)
        if (r + step < nrow && first_s[r + step] <= p) r += step;
      unsigned long long m = mask_s[r];
      for (int t = p - first_s[r]; t > 0; --t) m &= m - 1;  // the t-th candidate of r
      const int c = __ffsll(static_cast<long long>(m)) - 1;
      const double* xr = rows_s + r * d;
      const double* mr = mu_s + c * d;
      double acc = 0.0;
      for (int j = 0; j < d; ++j) {
        const double diff = __dsub_rn(xr[j], mr[j]);
        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
      }
      dist_s[p] = acc;
    }
    __syncthreads();
    for (int r = tid; r < nrow; r += kResThreads) {
      double best = 1e300;
      int bi = 0;
      unsigned long long m = mask_s[r];
      for (int p = first_s[r]; p < first_s[r + 1]; ++p) {
        const int c = __ffsll(static_cast<long long>(m)) - 1;
        m &= m - 1;
        if (dist_s[p] < best) {
          best = dist_s[p];
          bi = c;
        }
      }
      a_s[r] = bi;
      if (assign) assign[idx_s[r]] = bi;
    }
    __syncthreads();
    if (jj < d) {  // fold rows in list order; thread (rr, jj) owns cells (c, jj), c % R == rr
      for (int r = 0; r < nrow; ++r) {
        const int a = a_s[r];
        if (a % R == rr) {
          sums_s[a * d + jj] += rows_s[r * d + jj];
          if (jj == 0) cnt_s[a] += 1;
        }
      }
    }
  }
  __syncthreads();
  double* ps = part_sums + static_cast<size_t>(blockIdx.x) * k * d;
  for (int e = tid; e < k * d; e += kResThreads) ps[e] = sums_s[e];
  for (int c = tid; c < k; c += kResThreads) part_counts[static_cast<size_t>(blockIdx.x) * k + c] = cnt_s[c];
}

}  // namespace sk

static int screened_grid(int64_t n) {
  const int64_t tiles = (n + sk::kTile - 1) / sk::kTile;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(tiles, sm_count())));
}

static long long pend_capacity(int64_t n, int grid) {
  const int64_t tiles = (n + sk::kTile - 1) / sk::kTile;
  return ((tiles + grid - 1) / grid) * sk::kTile;
}

struct ScreenedWs {
  long long* pend_count;
  long long* part_counts;  // [(1+kResSplit)*grid][k]: main kernel, then resolve kernel
  double* part_sums;       // [(1+kResSplit)*grid][k*d]
  long long* pend_idx;     // [grid][cap]
  unsigned long long* pend_mask;
  size_t used;
};

static ScreenedWs carve_screened(void* base, int64_t n, int d, int k, int grid) {
  const long long cap = pend_capacity(n, grid);
  Carve c(base);
  ScreenedWs w;
  w.pend_count = c.take<long long>(grid);
  const int parts = (1 + sk::kResSplit) * grid;
  w.part_counts = c.take<long long>(static_cast<size_t>(parts) * k);
  w.part_sums = c.take<double>(static_cast<size_t>(parts) * k * d);
  w.pend_idx = c.take<long long>(static_cast<size_t>(grid) * cap);
  w.pend_mask = c.take<unsigned long long>(static_cast<size_t>(grid) * cap);
  w.used = c.used;
  return w;
}

size_t kmeans_screened_workspace_bytes(int64_t n, int d, int k) {
  if (d < 2 || d > sk::kMaxD || (d & 1) || k < 1 || k > sk::kMaxK) return 0;
  return carve_screened(nullptr, n, d, k, screened_grid(n)).used + 256;
}

int kmeans_screened_step(const double* x, int64_t n, int d, int k, const double* mu,
                         int32_t* assign, long long* counts, double* sums, void* ws,
                         size_t ws_bytes, cudaStream_t stream, bool probe_only) {
  DLX_REQUIRE(d >= 2 && d <= sk::kMaxD && (d & 1) == 0 && k >= 1 && k <= sk::kMaxK,
              DLX_ERR_GENERATION,
              "GenerationFailed: screened k-means needs even d <= %d and k <= %d (got d=%d k=%d)",
              sk::kMaxD, sk::kMaxK, d, k);
  DLX_REQUIRE((reinterpret_cast<uintptr_t>(x) & 15) == 0, DLX_ERR_GENERATION,
              "GenerationFailed: screened k-means needs 16-byte aligned samples");
  if (probe_only) return DLX_OK;
  const int grid = screened_grid(n);
  const long long cap = pend_capacity(n, grid);
  ScreenedWs w = carve_screened(ws, n, d, k, grid);
  DLX_REQUIRE(ws && w.used <= ws_bytes, DLX_ERR_ARG, "k-means workspace too small (%zu < %zu)",
              ws_bytes, w.used);
  DLX_CUDA(cudaFuncSetAttribute(sk::kmeans_screened_kernel,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sk::kSmemBytes)));
  static const bool tracing = getenv("DLX_KMEANS_TRACE") != nullptr;
  long long* trace = nullptr;
  if (tracing) DLX_CUDA(cudaMalloc(&trace, sizeof(long long) * grid * 40));
  sk::kmeans_screened_kernel<<<grid, sk::kThreads, sk::kSmemBytes, stream>>>(
      x, n, d, k, mu, assign, w.part_counts, w.part_sums, w.pend_idx, w.pend_mask, w.pend_count, cap,
      trace);
  DLX_LAUNCHED("kmeans_screened_kernel");
  if (tracing) {  // debug only: per-role cycle split averaged over CTAs
    std::vector<long long> h(static_cast<size_t>(grid) * 40);
    DLX_CUDA(cudaStreamSynchronize(stream));
    DLX_CUDA(cudaMemcpy(h.data(), trace, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
    cudaFree(trace);
    const char* names[5] = {"producer", "mma", "convert", "epilogue", "fold"};
    for (int r = 0; r < 5; ++r) {
      double avg[8] = {0};
      for (int b = 0; b < grid; ++b)
        for (int i = 0; i < 8; ++i) avg[i] += static_cast<double>(h[(static_cast<size_t>(b) * 5 + r) * 8 + i]) / grid;
      fprintf(stderr, "[dlx trace] %-9s", names[r]);
      for (int i = 0; i < 8; ++i) fprintf(stderr, " %10.0f", avg[i]);
      fprintf(stderr, "\n");
    }
  }
  const size_t rsmem =
      (static_cast<size_t>(2 * k + sk::kResChunk) * d + sk::kResMaxPairs) * sizeof(double);
  DLX_CUDA(cudaFuncSetAttribute(sk::kmeans_resolve_kernel,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(rsmem)));
  sk::kmeans_resolve_kernel<<<grid * sk::kResSplit, sk::kResThreads, rsmem, stream>>>(
      x, d, k, mu, assign, w.pend_idx, w.pend_mask, w.pend_count, cap,
      w.part_counts + static_cast<size_t>(grid) * k, w.part_sums + static_cast<size_t>(grid) * k * d);
  DLX_LAUNCHED("kmeans_resolve_kernel");
  return kmeans_finalize(w.part_counts, w.part_sums, (1 + sk::kResSplit) * grid, k, d, counts, sums,
                         stream);
}

// pending (re-checked) samples of the last screened step on this workspace
int kmeans_screened_pending(const void* ws, int64_t n, int d, int k, int64_t* out, cudaStream_t stream) {
  const int grid = screened_grid(n);
  std::vector<long long> h(grid);
  DLX_CUDA(cudaMemcpyAsync(h.data(), ws, sizeof(long long) * grid, cudaMemcpyDeviceToHost, stream));
  DLX_CUDA(cudaStreamSynchronize(stream));
  long long s = 0;
  for (long long v : h) s += v;
  *out = s;
  (void)d;
  (void)k;
  return DLX_OK;
}

}  // namespace dlx

extern "C" int dlx_kmeans_last_recheck_count(const void* d_workspace, int64_t n, int32_t d,
                                             int32_t k, int64_t* h_count, dlx_stream_t stream) {
  DLX_REQUIRE(d_workspace && h_count, DLX_ERR_ARG, "recheck count: null argument");
  return dlx::kmeans_screened_pending(d_workspace, n, d, k, h_count, stream);
}
