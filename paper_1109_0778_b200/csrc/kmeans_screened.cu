// kmeans_screened.cu — the k-means fused multiloop with a tcgen05 integer distance screen, an
// exact fp64 recheck, and the bucket-reduce as an exact integer one-hot GEMM on the same
// tensor cores.  Assignments stay bit-identical to the reference argmin chain
// (proj/src/stage.cpp:73-104 staged_if chain over the inner mk_reduce distances,
// loops.cpp:111-174); per-centroid sums are exact fixed-point sums rounded once.
//
// Why a screen: the direct form costs 3*N*k*d fp64 ops (2.1e11 per C4 iteration, ~11 ms at
// the FP64 pipe peak) against 1.34 ms of HBM time.  argmin_c (x-mu_c)^2 =
// argmin_c (|mu_c|^2 - 2 x.mu_c), and x.mu_c is a GEMM.  We compute it EXACTLY on integer
// tensor cores for 23-bit fixed-point copies of x and mu, bound the fixed-point error
// rigorously, and only re-evaluate the reference's own fp64 chain where the bound cannot
// separate the best centroid from the others.
//
// Fixed point.  Per launch e_m with |mu| < 2^e_m over finite centroids and e_t = e_m + 1.
// Each sample element becomes the 64-bit word
//   Z'' = floor(x * 2^(62-e_t)) + 2^63 + 2^39           (unsigned; bytes b7 .. b0)
// computed with three directed-rounding fp64 fmas (floor(x*2^(30-e_t)) and the floor of the
// remainder * 2^32).  Its top 24 bits are X'' = 2^23 + X with X = rint(x * 2^(22-e_t)) (+-2^-40),
// so the screen reads the planes h'' = b7, l = b6, F = b5 (all u8) and mu is split as before:
// M = rint(mu * 2^(22-e_m)) = 65536 h' + 256 l' + G (h' s8; l', G u8).  tcgen05.mma kind::i8
// computes exact int32 accumulators
//   HH = sum h'' h',  CR = sum (h'' l' + l h'),  W1 = sum (h'' G + F h' + l l'),  W2 = sum (l G + F l')
// so sum X'' M = 2^32 HH + 2^24 CR + 2^16 W1 + 2^8 W2 + sum F G (the last term, in
// [0, d*255^2], is dropped).  Q'' = 256 HH + CR + (W1>>8) + (W2>>16) satisfies
// sum X'' M / 2^24 in [Q'', Q'' + 2.25], and sum X M = sum X'' M - 2^23 sum_j M_j.  In units
// U = 2^(e_t+e_m-20) the score T_c = floor(|mu_c|^2/U) + sum_j M_cj - 2 Q''_c brackets
// |mu_c|^2/U - 2 x.mu_c/U within [T_c - 4.5 - 2e, T_c + 1 + 2e], e = ((sum|X| + sum|M|)/2 +
// d/4 + 2^-40 sum|M|)/2^24, and the reference's fp64 chain differs from the real distance by
// < 1 unit (|e_m| <= 400).  So every centroid with T_c > min_c T_c + W, W = 10 + ceil(4e),
// has a strictly larger reference distance than some other centroid and cannot be the
// argmin.  One survivor => it IS the reference argmin.  Several survivors => the sample goes
// to the pending list and is re-evaluated with the reference chain (sequential j, no FMA,
// strict <, ascending c, start (1e300, 0)).  Rows with |x| >= 2^e_t, inf or NaN send the
// sample to the exact chain over every centroid.  NaN / inf centroids never win the chain
// and are excluded from the screen.
//
// Three accumulators (the default, DLX_KMEANS_SCREEN_ACC=3).  The TMEM read-out of the screen
// accumulators (128 lanes x 4 B per column) is the epilogue's floor per tile, so W2 is not
// accumulated: 0 <= W2_c <= 255 sum_j (l'_cj + G_cj) =: 2^16 beta_c, and with
// Q3 = 256 HH + CR + (W1>>8) the score T3_c = nm_c - 2 Q3_c brackets the distance within
// [T3_c - 4.5 - 2 beta_c - 2e, T3_c + 1 + 2e]: window W3 = W + 2 ceil(max_c beta_c).  Rows with
// several W3-survivors (~0.2 % on uniform data, against ~0.07 % for W) are refined in the
// epilogue before they count as pending: their W2_c for the survivors only is summed exactly
// from the sample's b6 / b5 planes (still in the plane buffer) and the centroid planes with
// dp4a, T4_c = T3_c - 2 (W2_c >> 16) is the four-accumulator score, and the survivors are
// re-screened with W (sound: every centroid outside the W3-survivors already lost).  So the
// pending rows are exactly those of the four-accumulator screen, and a quarter of the TMEM
// read-out (and its W2 arithmetic) is gone from every row.
//
// Bucket-reduce.  The eight planes of a 128-sample tile are stored as four SW128 buffers of
// 128-byte rows [b7|b6], [b5|b4], [b3|b2], [b1|b0] (row = sample).  Read K-major they are the
// screen's A operand; read MN-major (M = plane x column, K = sample) the SAME bytes are the A
// operand of D[(plane, j)][c] += sum_q plane(x_qj) * onehot(a_q == c), whose B operand is the
// tile's one-hot assignment matrix (MN-major [q][c]).  The int32 accumulators live in TMEM
// for the whole launch (<= 128*255 per tile, < 2^31 for up to 65,793 tiles per CTA), so the
// per-centroid sums sum_q Z''_q = sum_p 2^(8p) D_p are EXACT integers, minus count_c *
// (2^63 + 2^39), times 2^(e_t-62), rounded once to fp64.  The fixed-point rounding is below
// 2^(e_t-62) per element; rows holding a nonzero |x| < 2^(e_t-30) (where that could exceed a
// 2^-32 relative error) take the exact fp64 fold with the re-checked samples.  The fold is
// order-free, hence deterministic.
//
// Kernel shape: one persistent CTA per SM (227 KiB smem: three 64 KiB plane buffers, the
// centroid planes, two one-hot buffers), 24 warps, warp-specialised around mbarriers:
//   warp 0      TMEM owner + screen MMA issuer: per tile 8 tcgen05.mma (N = 64/192/128/128,
//               centroid planes concatenated along N) into 4 x 64 int32 screen columns
//   warp 1      fold MMA issuer: per tile 16 MN-major tcgen05.mma into the persistent 4 x 64
//               fold columns; its commits free the plane and one-hot buffers
//   warp 2      tail: assignment stores, per-centroid counts, the ordered pending list
//   warps 4-7   epilogue (TMEM lane quarters): tcgen05.ld the screen columns, scores, minimum,
//               survivor mask (funnel-shifted sign bits), decision, the tile's one-hot rows;
//               at the end the exact fold flush
//   warps 8-23  converters: 32-byte row loads a whole tile ahead in registers, Z via one
//               round-down fma + F2I.S64, byte-plane transposes (PRMT), conflict-free STS
//   registers   80 at launch, rebalanced by setmaxnreg: warps 0-3 32, epilogue 128, converters 80
//   re-checks   after the CTA's last tile the epilogue warps evaluate the reference chain for
//               the pending samples (one thread per (sample, candidate) pair), write their
//               assignments and fold their rows into the CTA's record in fp64, in list order.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "sm100.cuh"

namespace dlx {

int kmeans_finalize(const long long* part_counts, const double* part_sums, int parts, int k, int d,
                    long long* counts, double* sums, cudaStream_t stream, double* mu_out);

namespace sk {

using namespace sm100;

constexpr int kTile = 128;   // samples per tile = MMA M
constexpr int kMaxD = 64;
constexpr int kMaxK = 64;
#ifndef DLX_KMEANS_CONV_WARPS
#define DLX_KMEANS_CONV_WARPS 16
#endif
constexpr int kNumC = DLX_KMEANS_CONV_WARPS;   // converter warps (kConvRows rows of every tile each)
constexpr int kConvRows = kTile / kNumC;
constexpr int kPairs = kConvRows / 2;                      // row pairs per converter warp per tile
constexpr int kBuf = kNumC == 8 ? kPairs : 4;             // rolling register buffer (pairs)
constexpr int kNumA = 3;     // plane buffers in flight
#ifndef DLX_KMEANS_L2_AHEAD
#define DLX_KMEANS_L2_AHEAD 3
#endif
constexpr int kL2Ahead = DLX_KMEANS_L2_AHEAD;   // converters' L2 prefetch distance (tiles; 0 = off)
#ifndef DLX_KMEANS_SCREEN_ACC
#define DLX_KMEANS_SCREEN_ACC 3
#endif
constexpr int kAcc = DLX_KMEANS_SCREEN_ACC;   // screen accumulators: 3 (HH, CR, W1; W2 refined) or 4
static_assert(kAcc == 3 || kAcc == 4, "screen accumulators");
// warpgroup 0: warp 0 screen MMAs, warp 1 fold MMAs, warp 2 tail (warp 3 idle); warpgroup 1:
// epilogue; then the converter warpgroups.  Registers are rebalanced with setmaxnreg after the
// prologue: warpgroup 0 drops to 32, the epilogue runs at 128, converters take the rest.
constexpr int kWarpMma = 0, kWarpFold = 1, kWarpTail = 2, kWarpE0 = 4, kWarpC0 = 8;
constexpr int kThreads = (kWarpC0 + kNumC) * 32;
constexpr int kRegsLaunch = (65536 / kThreads) & ~7;
constexpr int kRegsIssuer = 32, kRegsEpi = 128;
constexpr int kRegsConvRaw = (kThreads * kRegsLaunch - 128 * kRegsIssuer - 128 * kRegsEpi) / (32 * kNumC);
constexpr int kRegsConv = (kRegsConvRaw > 248 ? 248 : kRegsConvRaw) & ~7;
static_assert(kNumC == 8 || kNumC == 16, "converter warps");
static_assert(kRegsConv >= kRegsLaunch || kRegsEpi >= kRegsLaunch, "register plan");
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kFoldCol = 256;                        // fold accumulators: columns 256..511
constexpr uint32_t kPlane2 = kTile * 128;                 // one [b_hi|b_lo] SW128 buffer, 16 KiB
constexpr uint32_t kABuf = 4 * kPlane2;                   // eight planes, 64 KiB
constexpr uint32_t kOffA = 0;
constexpr uint32_t kOffB = kOffA + kNumA * kABuf;         // centroid planes: rows [h'' | l' | G], 192 x 64 B, SW64
constexpr uint32_t kOffOH = kOffB + 3 * kMaxK * 64;       // one-hot [q][c] 128 x 64 B, SW64, x2
constexpr uint32_t kOHBuf = kTile * 64;
constexpr uint32_t kOffMisc = kOffOH + 2 * kOHBuf;
static_assert(kOffA % 1024 == 0 && kOffB % 1024 == 0 && kOffOH % 512 == 0,
              "UMMA operand alignment");
static_assert(kNumA * kABuf >= 2u * kMaxK * 64 * 16, "final fold scratch must fit the plane buffers");
constexpr double kMagic = 6755399441055744.0;        // 1.5 * 2^52: x + kMagic rounds x to an integer
constexpr int kFoldBits = 30;  // rows with a nonzero |x| < 2^(e_t - 30) take the exact fp64 fold

struct Misc {
  uint64_t a_full[kNumA], c_full[kNumA], a_empty[kNumA], oh_full[2], oh_empty[2];
  uint64_t t_full, t_empty, fold_done;
  unsigned long long valid;
  uint32_t tmem_base;
  int em, yabs, disabled, window, window4, bsum_max;   // window4: W; window: W (4 acc) or W3
  uint32_t mu_maxhi;
  alignas(16) int nm0[kMaxK];             // floor(|mu_c|^2 / U) + sum_j M_cj
  double nmf[kMaxK];
  int cnt[kMaxK];                         // screened rows folded per centroid (this CTA)
  alignas(16) unsigned char rowflag[kNumA][kTile];  // 1: exact chain over every centroid; 2: exact fold
  int pcount[2][4];
  uint64_t dec_full[2], dec_empty[2];
  int dec_a[2][kTile];                    // per row: assigned centroid (screened), -1 pending, -2 padding
  unsigned long long dec_mask[2][kTile];  // candidate mask of pending rows
};
constexpr uint32_t kSmemBytes = kOffMisc + sizeof(Misc);
static_assert(kSmemBytes <= 232448, "shared-memory plan exceeds 227 KiB");
constexpr int kTraceTiles = 64;
constexpr int kInvalidNm = 0x70000000;  // > any valid score (|T| < 1.4e9)
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

// streaming 32-byte / 16-byte loads of sample rows (read once: no L1 allocation)
__device__ __forceinline__ void ldg256(const double* p, double& a, double& b, double& c, double& d) {
  asm("ld.global.nc.L1::no_allocate.L2::256B.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
__device__ __forceinline__ void ldg128(const double* p, double& a, double& b) {
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "l"(p));
}

// Rows of tile t: global row of tile row q is row0 + q, valid for q in [qlo, qhi).  With kShift
// (n >= kTile) the last tile is moved back to end at row n, so every tile is a full, unclamped
// 128-row block; its first qlo rows repeat rows of the previous tile and are ignored.
struct TileRows {
  int64_t row0;
  int qlo, qhi;
};
template <bool kShift>
__device__ __forceinline__ TileRows tile_rows(int64_t t, int64_t n) {
  const int64_t start = t * kTile;
  if (kShift && start + kTile > n) return {n - kTile, static_cast<int>(start - (n - kTile)), kTile};
  return {start, 0, static_cast<int>(n - start < kTile ? n - start : kTile)};
}

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok) : "r"(smem_addr(bar)), "r"(parity) : "memory");
  return ok != 0;
}

// 1: |x| >= 2^e_t, inf or NaN (screen out of range); 2: 0 < |x| < 2^(e_t - 30) (fold precision)
__device__ __forceinline__ int elem_flag(double x, uint32_t hw_hi, uint32_t hw_lo) {
  const uint32_t hw = static_cast<uint32_t>(__double2hiint(x)) & 0x7fffffffu;
  const uint32_t lw = static_cast<uint32_t>(__double2loint(x));
  return (hw >= hw_hi ? 1 : 0) | ((hw < hw_lo && (hw | lw) != 0u) ? 2 : 0);
}

constexpr int kResChunk = 64;
template <int NT, class Sync>
__device__ __forceinline__ void resolve_list(int tid, Sync sync, const double* __restrict__ x, int d,
                                             const double* __restrict__ mu_s, int32_t* __restrict__ assign,
                                             const long long* __restrict__ pidx,
                                             const unsigned long long* __restrict__ pmask, long long lo,
                                             long long hi, double* sums_s, long long* cnt_s, double* rows_s,
                                             double* dist_s, long long* idx_s, unsigned long long* mask_s,
                                             int* first_s, int* a_s, long long* tr = nullptr);

template <int kD, bool kWide>
__global__ void __launch_bounds__(kThreads, 1)
kmeans_screened_kernel(const double* __restrict__ x, int64_t n, int d, int k,
                       const double* __restrict__ mu, int32_t* __restrict__ assign,
                       long long* __restrict__ part_counts, double* __restrict__ part_sums,
                       long long* __restrict__ pend_idx, unsigned long long* __restrict__ pend_mask,
                       long long* __restrict__ pend_count, long long pend_cap,
                       long long* __restrict__ trace) {
  // optional per-tile event clocks (build with -DDLX_KMEANS_TRACE, run with DLX_KMEANS_TRACE=1):
  // trace[(cta * kTraceTiles + m) * 8 + event]
#ifdef DLX_KMEANS_TRACE
#define TRACE_PH(ev) do { if (trace) trace[(static_cast<size_t>(blockIdx.x) * kTraceTiles + kTraceTiles - 1) * 16 + (ev)] = clock64(); } while (0)
#define TRACE_EV(m, ev) do { if (trace && (m) < kTraceTiles - 1) trace[(static_cast<size_t>(blockIdx.x) * kTraceTiles + (m)) * 16 + (ev)] = clock64(); } while (0)
#else
#define TRACE_EV(m, ev) do { } while (0)
#define TRACE_PH(ev) do { } while (0)
#endif
  extern __shared__ __align__(1024) unsigned char smem[];
  Misc& S = *reinterpret_cast<Misc*>(smem + kOffMisc);
  if (threadIdx.x == 0) TRACE_PH(0);
  constexpr bool kShift = kD == 64;   // the host launches the d = 64 variant only for n >= kTile
  unsigned char* Bm = smem + kOffB;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t ntiles = (n + kTile - 1) / kTile;
  const int mtiles = static_cast<int>((ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x);

  // ---- prologue: barriers, B operands (fixed-point centroids), per-centroid constants ------
  if (tid == 0) {
    for (int s = 0; s < kNumA; ++s) {
      mbar_init(&S.a_full[s], kNumC);
      mbar_init(&S.c_full[s], kNumC);
      mbar_init(&S.a_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&S.oh_full[s], 4);
      mbar_init(&S.oh_empty[s], 1);
    }
    for (int s2 = 0; s2 < 2; ++s2) {
      mbar_init(&S.dec_full[s2], 4);
      mbar_init(&S.dec_empty[s2], 1);
    }
    mbar_init(&S.t_full, 1);
    mbar_init(&S.t_empty, 4);
    mbar_init(&S.fold_done, 1);
    S.valid = 0;
    S.yabs = 0;
    S.mu_maxhi = 0;
    S.bsum_max = 0;
    fence_mbar_init();
  }
  if (tid < kMaxK) S.cnt[tid] = 0;
  // launched with programmatic dependent launch: everything above overlaps the previous
  // kernel (the centroid update); from here on we read what it wrote
  pdl_wait();
  pdl_trigger();
  // centroids into shared memory (the plane buffers are free until the first conversion), one
  // coalesced pass; then one warp per centroid
  double* mu_s = reinterpret_cast<double*>(smem + kOffA);   // [c][64]
  for (int e = tid; e < k * d; e += kThreads) {
    const int c = e / d, j = e - c * d;
    mu_s[c * kMaxD + j] = __ldg(mu + e);
  }
  __syncthreads();
  for (int c = warp; c < kMaxK; c += kThreads / 32) {  // validity (all finite), max |mu| high word, |mu|^2
    uint32_t mx = 0;
    bool ok = c < k;
    double nm = 0.0;
    if (ok) {
      for (int j = lane; j < d; j += 32) {
        const double v = mu_s[c * kMaxD + j];
        const uint32_t hw = static_cast<uint32_t>(__double2hiint(v)) & 0x7fffffffu;
        if (hw >= 0x7ff00000u) ok = false;
        mx = max(mx, hw);
        nm += v * v;   // any summation order: |mu|^2 enters the bound through floor(.) with a unit of margin
      }
      ok = __all_sync(0xffffffffu, ok);
      mx = __reduce_max_sync(0xffffffffu, mx);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nm += __shfl_xor_sync(0xffffffffu, nm, o);
    }
    if (lane == 0) {
      S.nmf[c] = nm;
      if (ok) {
        atomicOr(&S.valid, 1ull << c);
        atomicMax(&S.mu_maxhi, mx);
      }
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
    for (int c = warp; c < kMaxK; c += kThreads / 32) {
      const bool cv = (valid >> c) & 1;
      int sa = 0, ssum = 0, sb = 0;
      for (int j = lane; j < kMaxD; j += 32) {
        // h'' = (Y >> 16) + 128 in [64, 192] (unsigned; the offset adds a per-sample constant to
        // every centroid's score); invalid centroids and columns past d are all-zero rows
        const bool live = cv && j < d;
        const int Y = live ? rint_magic(mu_s[c * kMaxD + j] * scale) : 0;
        Bm[sw64_offset(c, j)] = static_cast<unsigned char>(live ? (Y >> 16) + 128 : 0);
        Bm[sw64_offset(64 + c, j)] = static_cast<unsigned char>(Y >> 8);
        Bm[sw64_offset(128 + c, j)] = static_cast<unsigned char>(Y);
        sa += abs(Y);
        ssum += Y;
        sb += ((Y >> 8) & 255) + (Y & 255);   // l'_cj + G_cj (zero for dead rows)
      }
      sa = __reduce_add_sync(0xffffffffu, sa);
      ssum = __reduce_add_sync(0xffffffffu, ssum);
      sb = __reduce_add_sync(0xffffffffu, sb);
      if (lane == 0) {
        if (cv) {
          atomicMax(&S.yabs, sa);
          atomicMax(&S.bsum_max, sb);
        }
        // per-launch score constants (the sample exponent is fixed at e_t = e_m + 1)
        S.nm0[c] = (S.disabled || !cv) ? kInvalidNm
                                       : __double2int_rd(S.nmf[c] * ldexp(1.0, 19 - 2 * S.em)) + ssum;
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    // W = 10 + ceil(4e), e = ((d*2^22 + max_c sum|M|)/2 + d/4) / 2^24  (+1 margin covers 2^-40 terms)
    const long long num = (static_cast<long long>(d) << 22) + S.yabs;
    S.window4 = 10 + static_cast<int>((2 * num + d + (1ll << 24) - 1) >> 24);
    // W3 = W + 2 ceil(beta_max), beta_c = 255 sum_j (l'_cj + G_cj) / 2^16 (W2 not accumulated)
    S.window = S.window4 + (kAcc == 3 ? 2 * static_cast<int>((255ll * S.bsum_max + 65535) >> 16) : 0);
  }
  fence_proxy_async_smem();
  if (warp == kWarpMma) tmem_alloc<kTmemCols>(&S.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;
  if (threadIdx.x == 0) TRACE_PH(1);

  if (warp < kWarpE0) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsIssuer));
  if (warp == kWarpMma) {
    // ======================= screen MMA issuer =======================
    // the whole warp runs the loop and waits (a converged warp sleeping in try_wait); lane 0
    // issues.  A lane-0-only loop left 31 lanes diverged at the exit barrier, and the issuer's
    // SMSP then ran its converters ~1K cycles per tile behind the idle-warp SMSP (trace r121-r123).
    {
      // all operands unsigned: sample planes h'' = b7, l = b6, F = b5; centroid rows h'', l', G
      constexpr uint32_t ID_64 = idesc_i8(kTile, 64, 0, 0), ID_128 = idesc_i8(kTile, 128, 0, 0);
      constexpr uint32_t ID_192 = idesc_i8(kTile, 192, 0, 0);
      const uint32_t bm = smem_addr(Bm);
      const int nk = (d + 31) / 32;
      for (int ns = 0; ns < mtiles; ++ns) {
        mbar_wait(&S.a_full[ns % kNumA], (ns / kNumA) & 1);
        TRACE_EV(ns, 8);
        if (ns >= 1) mbar_wait(&S.t_empty, (ns - 1) & 1);
        TRACE_EV(ns, 9);
        tc_fence_after();
        const uint32_t a0 = smem_addr(smem + kOffA + (ns % kNumA) * kABuf);
        if (lane == 0) {
        for (int kk = 0; kk < nk; ++kk) {
          const uint64_t xh = sw128_kmajor_desc(a0 + 32 * kk);             // b7 = h''
          const uint64_t xl = sw128_kmajor_desc(a0 + 64 + 32 * kk);        // b6 = l
          const uint64_t xf = sw128_kmajor_desc(a0 + kPlane2 + 32 * kk);   // b5 = F
          const uint64_t m0 = sw64_kmajor_desc(bm + 32 * kk);              // rows h'', l', G
          const uint64_t m1 = sw64_kmajor_desc(bm + 64 * 64 + 32 * kk);    // rows l', G
          const uint32_t acc = kk > 0;
          // TMEM columns: HH 0-63, CR 64-127, W1 128-191 (, W2 192-255)
          mma_i8(tmem + 0, xh, m0, ID_64, acc);      // HH  = h'' h''
          if constexpr (kAcc == 4) {
            mma_i8(tmem + 64, xl, m0, ID_192, acc);  // CR += l h'',  W1 += l l',  W2 += l G
            mma_i8(tmem + 64, xh, m1, ID_128, 1);    // CR += h'' l', W1 += h'' G
            mma_i8(tmem + 128, xf, m0, ID_128, 1);   // W1 += F h'',  W2 += F l'
          } else {
            mma_i8(tmem + 64, xl, m0, ID_128, acc);  // CR += l h'',  W1 += l l'
            mma_i8(tmem + 64, xh, m1, ID_128, 1);    // CR += h'' l', W1 += h'' G
            mma_i8(tmem + 128, xf, m0, ID_64, 1);    // W1 += F h''
          }
        }
        mma_commit(&S.t_full);
        TRACE_EV(ns, 0);
        }
        __syncwarp();
      }
    }
  } else if (warp == kWarpFold) {
    // ======================= fold MMA issuer =======================
    {   // converged warp, lane 0 issues (as the screen issuer)
      constexpr uint32_t ID_fold = idesc_i8_major(kTile, 64, 0, 0, 1, 1);
      for (int nf = 0; nf < mtiles; ++nf) {
        mbar_wait(&S.oh_full[nf & 1], (nf >> 1) & 1);
        TRACE_EV(nf, 13);
        tc_fence_after();
        const uint32_t a0 = smem_addr(smem + kOffA + (nf % kNumA) * kABuf);
        const uint32_t oh = smem_addr(smem + kOffOH + (nf & 1) * kOHBuf);
        if (lane == 0) {
#pragma unroll
        for (int kk = 0; kk < kTile / 32; ++kk) {
          const uint64_t bdesc = sw64_kmajor_desc(oh + kk * 2048);   // MN-major [q][c], SW64
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const uint64_t adesc = sw128_kmajor_desc(a0 + g * kPlane2 + kk * 4096);  // MN-major
            mma_i8(tmem + kFoldCol + 64 * g, adesc, bdesc, ID_fold, (nf > 0 || kk > 0) ? 1u : 0u);
          }
        }
        mma_commit(&S.a_empty[nf % kNumA]);
        mma_commit(&S.oh_empty[nf & 1]);
        TRACE_EV(nf, 1);
        }
        __syncwarp();
      }
      if (lane == 0) mma_commit(&S.fold_done);
      __syncwarp();
    }
  } else if (warp == kWarpTail) {
    // ======================= tail: assignments, counts, pending list =======================
    // Off the critical path: consumes the epilogue's per-row decisions tile by tile, writes the
    // screened assignments, counts them per centroid, and appends the pending rows to this
    // CTA's list in row order (deterministic).
    long long* my_pidx = pend_idx + static_cast<size_t>(blockIdx.x) * pend_cap;
    unsigned long long* my_pmask = pend_mask + static_cast<size_t>(blockIdx.x) * pend_cap;
    long long pending = 0;
    for (int m = 0; m < mtiles; ++m) {
      const int64_t t = blockIdx.x + static_cast<int64_t>(m) * gridDim.x;
      const int64_t row0 = tile_rows<kShift>(t, n).row0;
      const int b = m & 1;
      mbar_wait(&S.dec_full[b], (m >> 1) & 1);
#pragma unroll 1
      for (int r0 = 0; r0 < kTile; r0 += 32) {
        const int r = r0 + lane;
        const int a = S.dec_a[b][r];
        if (a >= 0) {
          if (assign) assign[row0 + r] = a;
          atomicAdd(&S.cnt[a], 1);
        }
        const unsigned pb = __ballot_sync(0xffffffffu, a == -1);
        if (a == -1) {
          const long long slot = pending + __popc(pb & ((1u << lane) - 1));
          my_pidx[slot] = row0 + r;
          my_pmask[slot] = S.dec_mask[b][r];
          // the exact re-check at the end of the launch gathers this row: keep it in L2
          const char* xr = reinterpret_cast<const char*>(x + (row0 + r) * d);
          for (int off = 0; off < d * 8; off += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(xr + off));
        }
        pending += __popc(pb);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.dec_empty[b]);
    }
    if (lane == 0) pend_count[blockIdx.x] = pending;
    named_bar_split(7, 160);   // met by the epilogue warps' barrier 7 below
  }
  } else if (warp >= kWarpC0) {
    if constexpr (kRegsConv > kRegsLaunch) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsConv));
    // ======================= converters (16 warps) =======================
    // Warp cw owns rows kConvRows*cw .. +kConvRows-1 of every tile as row pairs (r, r + 4) of an
    // 8-row SW128 atom.  Lane (hl, p) = (lane >> 4, lane & 15) holds columns 4p .. 4p+3 of row
    // r + 4 hl: one coalesced 32-byte load per pair, issued kBuf pairs ahead into a rolling
    // register buffer (with kPairs = kBuf = 4: a whole tile ahead).  Rows r and r + 4 land in
    // disjoint bank halves, so every plane store is one wavefront.
    const int cw = warp - kWarpC0;
    const int D = kD ? kD : d;
    const int em = S.em, disabled = S.disabled;
    const int et = em + 1;
    const double s_hi = disabled ? 0.0 : ldexp(1.0, 30 - et);
    const double s_z = disabled ? 0.0 : ldexp(1.0, 62 - et);   // Z = floor(x * 2^(62 - e_t)), exact product
    const uint32_t hw_hi = static_cast<uint32_t>(1023 + et) << 20;          // |x| >= 2^e_t, inf, NaN
    const int lo_e = 1023 + et - kFoldBits;
    const uint32_t hw_lo = lo_e > 0 ? static_cast<uint32_t>(lo_e) << 20 : 0u;  // nonzero |x| < 2^(e_t-30)
    const int hl = lane >> 4, p = lane & 15;
    const int col0 = 4 * p;
    const int nvalid = col0 + 4 <= D ? 4 : (col0 + 2 <= D ? 2 : 0);
    // load column of this lane (clamped into the row) and the offset of its second pair
    const int lcol = nvalid ? col0 : 0;
    const int lcol2 = nvalid == 4 ? 2 : 0;
    const int rbase = kConvRows * cw + 4 * hl;   // tile row of this lane's pair 0
    auto pair_row = [](int i) { return 8 * (i >> 2) + (i & 3); };   // row offset of pair i
    // plane-store offset of pair i: soff[i & 3] + (i >> 2) * 1024
    uint32_t soff[4];
#pragma unroll
    for (int r4 = 0; r4 < 4; ++r4)
      soff[r4] = static_cast<uint32_t>(kConvRows / 8 * cw) * 1024u + static_cast<uint32_t>(r4 + 4 * hl) * 128u +
                 (((static_cast<uint32_t>(p >> 2) ^ (4u * hl)) ^ static_cast<uint32_t>(r4)) << 4) + 4u * (p & 3);
    double v[kBuf][4];
    auto tile_of = [&](int mm) { return static_cast<int64_t>(blockIdx.x) + static_cast<int64_t>(mm) * gridDim.x; };
    // unconditional loads from clamped addresses (the loaded registers need no phi copies,
    // which would wait on a load right after issuing it)
    auto load_pair = [&](const double* base, int64_t rows, int i, double (&dst)[4]) {
      int off = pair_row(i);
      if constexpr (!kShift) {
        if (rbase + off >= rows) off = static_cast<int>(rows - 1) - rbase;   // padding rows repeat the last row
      }
      const double* src = base + off * D;
      if constexpr (kWide) {
        ldg256(src, dst[0], dst[1], dst[2], dst[3]);
      } else {
        ldg128(src, dst[0], dst[1]);
        ldg128(src + lcol2, dst[2], dst[3]);
      }
    };
    auto base_of = [&](int mm, int64_t& rows) {
      const TileRows tr = tile_rows<kShift>(tile_of(mm), n);
      rows = tr.qhi;
      return x + (tr.row0 + rbase) * D + lcol;
    };
    int64_t cur_rows = 0;
    const double* cur = base_of(0, cur_rows);
    if (mtiles > 0) {
#pragma unroll
      for (int i = 0; i < kBuf; ++i) load_pair(cur, cur_rows, i, v[i]);
    }
    for (int m = 0; m < mtiles; ++m) {
      const int b = m % kNumA;
      int64_t nxt_rows = 0;
      const double* nxt = base_of(m + 1 < mtiles ? m + 1 : m, nxt_rows);
#if DLX_KMEANS_L2_AHEAD > 0
      // this warp's rows of tile m + kL2Ahead (contiguous) into L2 ahead of the register loads
      // (issued one tile ahead): those then wait on L2 rather than on HBM latency under load
      if (lane == 0 && m + kL2Ahead < mtiles) {
        const TileRows tp = tile_rows<kShift>(tile_of(m + kL2Ahead), n);
        const int64_t r0 = tp.row0 + kConvRows * cw;
        if (r0 + kConvRows <= n) bulk_prefetch_l2(x + r0 * D, static_cast<uint32_t>(kConvRows * D * 8));
      }
#endif
      if (cw == 0 && lane == 0) TRACE_EV(m, 2);
      if (m >= kNumA) mbar_wait(&S.a_empty[b], ((m / kNumA) - 1) & 1);
      if (cw == 0 && lane == 0) TRACE_EV(m, 3);
      unsigned char* Ab = smem + kOffA + b * kABuf;
      // conservative range test over the lane's values (exact row classification below, only
      // if some lane saw a value outside [2^(e_t-30), 2^e_t), zeros included); columns past d
      // hold copies and are not tested
      uint32_t mx = 0, mn = 0xffffffffu;
#pragma unroll
      for (int i = 0; i < kPairs; ++i) {
        double (&w)[4] = v[i % kBuf];
        uint32_t H[4], L[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t hw = static_cast<uint32_t>(__double2hiint(w[e])) & 0x7fffffffu;
          if (kD == 64 || e < nvalid) {
            mx = max(mx, hw);
            mn = min(mn, hw);
          }
          // Z + 2^39 = floor(x s + 2^39): one round-down fma (exact floor) + F2I.S64.FLOOR; the
          // + 2^63 is the top-bit flip applied to the b7 plane below
          const long long z = __double2ll_rd(__fma_rd(w[e], s_z, 549755813888.0));
          H[e] = static_cast<uint32_t>(static_cast<unsigned long long>(z) >> 32);
          L[e] = static_cast<uint32_t>(z);
        }
        if (i + kBuf < kPairs) load_pair(cur, cur_rows, i + kBuf, w);
        else load_pair(nxt, nxt_rows, i + kBuf - kPairs, w);
        // 4x4 byte transposes: plane word = that byte of the four consecutive columns
        const uint32_t ha = __byte_perm(H[0], H[1], 0x5140), hb = __byte_perm(H[0], H[1], 0x7362);
        const uint32_t hc = __byte_perm(H[2], H[3], 0x5140), hd = __byte_perm(H[2], H[3], 0x7362);
        const uint32_t la = __byte_perm(L[0], L[1], 0x5140), lb = __byte_perm(L[0], L[1], 0x7362);
        const uint32_t lc = __byte_perm(L[2], L[3], 0x5140), ld = __byte_perm(L[2], L[3], 0x7362);
        unsigned char* A0 = Ab + soff[i & 3] + (i >> 2) * 1024;
        unsigned char* A1 = Ab + (soff[i & 3] ^ 64u) + (i >> 2) * 1024;
        *reinterpret_cast<uint32_t*>(A0) = __byte_perm(hb, hd, 0x7632) ^ 0x80808080u;    // b7
        *reinterpret_cast<uint32_t*>(A1) = __byte_perm(hb, hd, 0x5410);                  // b6
        *reinterpret_cast<uint32_t*>(A0 + kPlane2) = __byte_perm(ha, hc, 0x7632);        // b5
        *reinterpret_cast<uint32_t*>(A1 + kPlane2) = __byte_perm(ha, hc, 0x5410);        // b4
        *reinterpret_cast<uint32_t*>(A0 + 2 * kPlane2) = __byte_perm(lb, ld, 0x7632);    // b3
        *reinterpret_cast<uint32_t*>(A1 + 2 * kPlane2) = __byte_perm(lb, ld, 0x5410);    // b2
        *reinterpret_cast<uint32_t*>(A0 + 3 * kPlane2) = __byte_perm(la, lc, 0x7632);    // b1
        *reinterpret_cast<uint32_t*>(A1 + 3 * kPlane2) = __byte_perm(la, lc, 0x5410);    // b0
      }
      cur = nxt;
      cur_rows = nxt_rows;
      const bool odd = disabled || ((kD == 64 || nvalid) && (mx >= hw_hi || mn < hw_lo));
      if (__any_sync(0xffffffffu, odd)) {
        // rare: classify row by row, re-reading this tile's values (the registers already hold
        // the next pairs)
        const TileRows tr = tile_rows<kShift>(tile_of(m), n);
#pragma unroll 1
        for (int i = 0; i < kPairs; ++i) {
          const int row = rbase + pair_row(i);
          int f = 0;
          if (row >= tr.qlo && row < tr.qhi)
            for (int e = 0; e < 4; ++e)
              if (col0 + e < d) f |= elem_flag(x[(tr.row0 + row) * d + col0 + e], hw_hi, hw_lo);
          const int f0 = static_cast<int>(__reduce_or_sync(0xffffffffu, static_cast<unsigned>(hl ? 0 : f)));
          const int f1 = static_cast<int>(__reduce_or_sync(0xffffffffu, static_cast<unsigned>(hl ? f : 0)));
          const int r = kConvRows * cw + pair_row(i);
          if (lane == 0) S.rowflag[b][r] = static_cast<unsigned char>(disabled ? 1 : (f0 & 1 ? 1 : f0));
          if (lane == 16) S.rowflag[b][r + 4] = static_cast<unsigned char>(disabled ? 1 : (f1 & 1 ? 1 : f1));
        }
      } else if (lane == 0) {
        static_assert(kConvRows == 8 || kConvRows == 16, "row-flag store width");
        if constexpr (kConvRows == 16)
          *reinterpret_cast<uint4*>(&S.rowflag[b][kConvRows * cw]) = make_uint4(0u, 0u, 0u, 0u);
        else
          *reinterpret_cast<uint2*>(&S.rowflag[b][kConvRows * cw]) = make_uint2(0u, 0u);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&S.a_full[b]);
        mbar_arrive(&S.c_full[b]);
        if (cw == 0) TRACE_EV(m, 4);
        if (cw == 7) TRACE_EV(m, 10);

      }
    }
  } else {
    if constexpr (kRegsEpi > kRegsLaunch) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsEpi));
    if constexpr (kRegsEpi < kRegsLaunch) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsEpi));
    // ======================= epilogue (4 warps, one per TMEM lane quarter) ===========
    const int quarter = warp & 3;
    const int q = quarter * 32 + lane;  // sample row within the tile (M row)
    const unsigned long long kmask = k == 64 ? ~0ull : ((1ull << k) - 1);
    const unsigned long long vmask = S.valid;   // finite centroids (the others never survive)
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    const int window = S.window;
    const int4* nm4 = reinterpret_cast<const int4*>(S.nm0);
    const uint32_t oh_row = (static_cast<uint32_t>(q) >> 3) * 512u + (q & 7) * 64u;
    const uint32_t oh_sw = (q & 7) >> 1;
    int oh_prev0 = -1, oh_prev1 = -1;   // chunk of this row's bit in each one-hot buffer's previous tile
    for (int m = 0; m < mtiles; ++m) {
      const int64_t t = blockIdx.x + static_cast<int64_t>(m) * gridDim.x;
      const int b = m & 1;
      const TileRows tr = tile_rows<kShift>(t, n);
      if (quarter == 0 && lane == 0) TRACE_EV(m, 5);
      mbar_wait(&S.t_full, m & 1);
      if (quarter == 0 && lane == 0) TRACE_EV(m, 6);
      tc_fence_after();
      int tv[64];
      int lmin = kInvalidNm;
#pragma unroll
      for (int ch = 0; ch < 8; ++ch) {
        const uint32_t col = 8 * ch;
        int hh[8], cr[8], w1[8], w2[8];
        tmem_ld8(tmem + lane_base + col, hh);
        tmem_ld8(tmem + lane_base + col + 64, cr);
        tmem_ld8(tmem + lane_base + col + 128, w1);
        if constexpr (kAcc == 4) tmem_ld8(tmem + lane_base + col + 192, w2);
        const int4 n0 = nm4[2 * ch], n1 = nm4[2 * ch + 1];
        const int nm[8] = {n0.x, n0.y, n0.z, n0.w, n1.x, n1.y, n1.z, n1.w};
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          // invalid centroids: zero B rows (Q = 0) and nm = kInvalidNm
          const int Q = hh[u] * 256 + cr[u] + (w1[u] >> 8) + (kAcc == 4 ? (w2[u] >> 16) : 0);
          const int v = nm[u] - 2 * Q;
          tv[8 * ch + u] = v;
          lmin = min(lmin, v);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.t_empty);
      if (quarter == 0 && lane == 0) TRACE_EV(m, 12);
      const int b3 = m % kNumA;
      mbar_wait(&S.c_full[b3], (m / kNumA) & 1);
      if (quarter == 0 && lane == 0) TRACE_EV(m, 11);
      unsigned long long full = 0;
      int hot = -2;   // -2 padding row, -1 pending, else the assigned centroid
      if (q >= tr.qlo && q < tr.qhi) {
        const int flag = S.rowflag[b3][q];
        bool pend = false;
        int a = -1;
        if (flag & 1) {
          full = kmask;  // |x| out of the screen's range, inf or NaN: the exact chain over all c
          pend = true;
        } else if (lmin < kNoCandidate) {
          // survivors tv[u] <= lmin + window: collect the sign bits of tv[u] - (lmin + window + 1)
          // with funnel shifts (valid scores of a row differ by < 2^30, so the signs are exact;
          // invalid centroids are masked out), then bit-reverse
          const int thr1 = lmin + window + 1;
          unsigned nlo = 0, nhi = 0;
#pragma unroll
          for (int u = 0; u < 32; ++u) nlo = __funnelshift_l(static_cast<unsigned>(tv[u] - thr1), nlo, 1);
#pragma unroll
          for (int u = 32; u < 64; ++u) nhi = __funnelshift_l(static_cast<unsigned>(tv[u] - thr1), nhi, 1);
          full = ((static_cast<unsigned long long>(__brev(nhi)) << 32) | __brev(nlo)) & vmask;
          if ((full & (full - 1)) == 0) {
            a = __ffsll(static_cast<long long>(full)) - 1;
          } else {
            pend = true;  // several survivors: resolved by the exact chain after the last tile
          }
        } else {
          a = 0;  // no finite centroid: the chain keeps its start index
        }
        if (flag & 2) pend = true;  // exact fp64 fold (the chain over the survivors re-derives a)
        hot = pend ? -1 : a;
      }
      // this tile's one-hot row q (MN-major [q][c], SW64); zero for pending / padding rows
      if (quarter == 0 && lane == 0) TRACE_EV(m, 14);
      if (m >= 2) mbar_wait(&S.oh_empty[b], ((m >> 1) - 1) & 1);
      if (quarter == 0 && lane == 0) TRACE_EV(m, 15);
      {
        unsigned char* ohb = smem + kOffOH + b * kOHBuf + oh_row;
#ifndef DLX_KMEANS_OH_FULL
        // only the 16-byte chunk that holds this row's bit now, and the one that held it in this
        // buffer's previous tile, change: after the first use of each buffer (all four chunks)
        // a row costs at most two stores
        const int nc = hot >= 0 ? (hot >> 4) : -1;
        const int pc = m >= 2 ? (b ? oh_prev1 : oh_prev0) : -2;
        if (b) oh_prev1 = nc;
        else oh_prev0 = nc;
        uint4 w = make_uint4(0u, 0u, 0u, 0u);
        if (nc >= 0) {
          const int rel = hot & 15;
          const uint32_t bit = 1u << (8 * (rel & 3));
          const int wi = rel >> 2;
          w.x = wi == 0 ? bit : 0u;
          w.y = wi == 1 ? bit : 0u;
          w.z = wi == 2 ? bit : 0u;
          w.w = wi == 3 ? bit : 0u;
        }
        if (pc == -2) {
#pragma unroll
          for (int ch = 0; ch < 4; ++ch)
            *reinterpret_cast<uint4*>(ohb + ((ch ^ oh_sw) << 4)) = ch == nc ? w : make_uint4(0u, 0u, 0u, 0u);
        } else {
          if (pc >= 0 && pc != nc) *reinterpret_cast<uint4*>(ohb + ((pc ^ oh_sw) << 4)) = make_uint4(0u, 0u, 0u, 0u);
          if (nc >= 0) *reinterpret_cast<uint4*>(ohb + ((nc ^ oh_sw) << 4)) = w;
        }
#else
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          uint4 w = make_uint4(0u, 0u, 0u, 0u);
          const int rel = hot - 16 * ch;
          const uint32_t bit = 1u << (8 * (rel & 3));
          if (rel >= 0 && rel < 16) {
            const int wi = rel >> 2;
            w.x = wi == 0 ? bit : 0u;
            w.y = wi == 1 ? bit : 0u;
            w.z = wi == 2 ? bit : 0u;
            w.w = wi == 3 ? bit : 0u;
          }
          *reinterpret_cast<uint4*>(ohb + ((ch ^ oh_sw) << 4)) = w;
        }
#endif
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.oh_full[b]);
      if (quarter == 0 && lane == 0) TRACE_EV(m, 7);
      // hand the decision to the tail warp
      if (m >= 2) mbar_wait(&S.dec_empty[b], ((m >> 1) - 1) & 1);
      S.dec_a[b][q] = hot;
      if (hot == -1) S.dec_mask[b][q] = full;   // read by the tail for pending rows only
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.dec_full[b]);
    }


    // ---- flush: exact per-centroid sums from the fold accumulators ------------------------
    // TMEM lane q < 64 holds planes b7, b5, b3, b1 of column j = q; lane 64 + j planes b6, b4,
    // b2, b0 (fold group g = columns 256 + 64 g).  Each thread forms its planes' partial sum
    // as an integer for every centroid into scratch (the plane buffers, free once every fold
    // MMA has completed); then every (c, j) cell adds the two halves, removes the per-row
    // offset count_c * (2^63 + 2^39) and scales by 2^(e_t - 62).
    mbar_wait(&S.fold_done, 0);
    if (q == 0) TRACE_PH(2);
    tc_fence_after();
    named_bar_split(7, 160);   // with the tail warp: every count is in S.cnt
    unsigned long long* scratch = reinterpret_cast<unsigned long long*>(smem + kOffA);
    {
      const int half = q >> 6, j = q & 63;
      for (int cc = 0; cc < 8; ++cc) {
        int acc[4][8];
#pragma unroll
        for (int g = 0; g < 4; ++g) tmem_ld8(tmem + lane_base + kFoldCol + 64 * g + 8 * cc, acc[g]);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          // planes 7-2g (half 0) or 6-2g (half 1): sum_g acc_g * 2^(8 (7 - 2g - half))
          unsigned __int128 s = 0;
#pragma unroll
          for (int g = 0; g < 4; ++g)
            s += static_cast<unsigned __int128>(static_cast<uint32_t>(acc[g][u])) << (8 * (7 - 2 * g - half));
          const int c = 8 * cc + u;
          unsigned long long* dst = scratch + 2 * ((half * kMaxK + c) * 64 + j);
          dst[0] = static_cast<unsigned long long>(s);
          dst[1] = static_cast<unsigned long long>(s >> 64);
        }
      }
    }
    tc_fence_before();
    named_bar(1, 128);
    // the record in shared memory (beyond the scratch), completed below by this CTA's own
    // pending rows, then written once
    double* sums_s = reinterpret_cast<double*>(smem + kOffA + 2 * kABuf);          // k*d
    {
      const int et = S.em + 1;
      const double unit = ldexp(1.0, et - 62);
      const unsigned __int128 off = (static_cast<unsigned __int128>(1) << 63) + (static_cast<unsigned __int128>(1) << 39);
      for (int e = q; e < kMaxK * 64; e += 128) {
        const int c = e >> 6, j = e & 63;
        if (c >= k || j >= d) continue;
        const unsigned long long* s0 = scratch + 2 * (c * 64 + j);
        const unsigned long long* s1 = scratch + 2 * ((kMaxK + c) * 64 + j);
        const unsigned __int128 hi = (static_cast<unsigned __int128>(s0[1]) << 64) | s0[0];
        const unsigned __int128 lo = (static_cast<unsigned __int128>(s1[1]) << 64) | s1[0];
        const __int128 tot = static_cast<__int128>(hi + lo - static_cast<unsigned __int128>(S.cnt[c]) * off);
        const long long th = static_cast<long long>(tot >> 64);
        const unsigned long long tl = static_cast<unsigned long long>(tot);
        const double v = __fma_rn(static_cast<double>(th), 18446744073709551616.0, static_cast<double>(tl));
        sums_s[c * d + j] = v * unit;
      }
    }
    if (q == 0) TRACE_PH(3);
    const long long npend = pend_count[blockIdx.x];   // written by the tail warp before barrier 7
    long long* cnt_s = reinterpret_cast<long long*>(smem + kOffOH);   // the one-hot buffers are free now
    if (npend > 0) {
      // resolve this CTA's pending rows in list order into the record (the chain over their
      // candidates, sequential j, no FMA; strict <; start (1e300, 0))
      for (int c = q; c < k; c += 128) cnt_s[c] = S.cnt[c];
      // the scratch is consumed: rows [64][d+1], distances, centroids [k][d+1] (padded strides)
      double* rows_s = reinterpret_cast<double*>(smem + kOffA);
      double* dist_s = rows_s + kResChunk * (kMaxD + 1);
      double* mu_s = dist_s + kResChunk * kMaxK;
      long long* idx_s = cnt_s + kMaxK;
      unsigned long long* mask_s = reinterpret_cast<unsigned long long*>(idx_s + kResChunk);
      int* first_s = reinterpret_cast<int*>(mask_s + kResChunk);
      int* a_s = first_s + kResChunk + 1;
      named_bar(1, 128);   // everyone is done reading the scratch
      {  // 16-byte loads, 8 per thread in flight
        const double2* mu2 = reinterpret_cast<const double2*>(mu);
        const int half = d / 2, total = k * half;
#pragma unroll 8
        for (int e = q; e < total; e += 128) {
          const int c = e / half, j2 = e - c * half;
          const double2 v = __ldg(mu2 + e);
          mu_s[c * (d + 1) + 2 * j2] = v.x;
          mu_s[c * (d + 1) + 2 * j2 + 1] = v.y;
        }
      }
      resolve_list<128>(q, [] { named_bar(1, 128); }, x, d, mu_s, assign,
                        pend_idx + static_cast<size_t>(blockIdx.x) * pend_cap,
                        pend_mask + static_cast<size_t>(blockIdx.x) * pend_cap, 0, npend, sums_s, cnt_s,
                        rows_s, dist_s, idx_s, mask_s, first_s, a_s,
                        trace ? trace + (static_cast<size_t>(blockIdx.x) * kTraceTiles + kTraceTiles - 1) * 16 + 8 : nullptr);
    } else {
      for (int c = q; c < k; c += 128) cnt_s[c] = S.cnt[c];
      named_bar(1, 128);
    }
    if (q == 0) TRACE_PH(4);
    double* ps = part_sums + static_cast<size_t>(blockIdx.x) * k * d;
    for (int e = q; e < k * d; e += 128) ps[e] = sums_s[e];
    for (int c = q; c < k; c += 128) part_counts[static_cast<size_t>(blockIdx.x) * k + c] = cnt_s[c];
  }
  __syncthreads();
  if (warp == kWarpMma) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
    if (lane == 0) TRACE_PH(5);
  }
}

// ---------------------------------------------------------------------------------------
// The exact re-check of one CTA's pending list [lo, hi), in chunks of kResChunk samples: the
// chunk's rows are gathered into shared memory next to the fp64 centroids, every (sample,
// candidate) pair is one thread's reference chain (sequential j, no FMA), each sample then
// merges its candidates in ascending centroid order (strict <, NaN never wins, start
// (1e300, 0)), and the rows are folded, in list order, into the record (sums_s, cnt_s) in
// shared memory (deterministic).  NT threads (tid in [0, NT)) synchronise with `sync`.
template <int NT, class Sync>
__device__ __forceinline__ void resolve_list(int tid, Sync sync, const double* __restrict__ x, int d,
                                             const double* __restrict__ mu_s, int32_t* __restrict__ assign,
                                             const long long* __restrict__ pidx,
                                             const unsigned long long* __restrict__ pmask, long long lo,
                                             long long hi, double* sums_s, long long* cnt_s, double* rows_s,
                                             double* dist_s, long long* idx_s, unsigned long long* mask_s,
                                             int* first_s, int* a_s, long long* tr) {
  constexpr int R = NT / 64;
#ifdef DLX_KMEANS_TRACE
  long long tacc[5] = {0, 0, 0, 0, 0}, t0 = clock64();
#define RTR(i) do { const long long _t = clock64(); tacc[i] += _t - t0; t0 = _t; } while (0)
#else
#define RTR(i) do { } while (0)
#endif
  const int jj = tid & 63, rr = tid >> 6;
  for (long long base = lo; base < hi; base += kResChunk) {
    const int nrow = static_cast<int>(hi - base < kResChunk ? hi - base : kResChunk);
    sync();
    for (int e = tid; e < nrow; e += NT) {
      idx_s[e] = pidx[base + e];
      mask_s[e] = pmask[base + e];
    }
    sync();
    RTR(0);
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
    {  // gather: 16-byte loads, up to 8 per thread in flight, into rows padded to stride d + 1
      const int half = d / 2, total = nrow * half;
      for (int e0 = tid; e0 < total; e0 += 8 * NT) {
        double2 v[8];
        int at[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * NT;
          at[u] = -1;
          if (e < total) {
            const int r = e / half, j2 = e - r * half;
            v[u] = __ldg(reinterpret_cast<const double2*>(x + idx_s[r] * d) + j2);
            at[u] = r * (d + 1) + 2 * j2;
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (at[u] >= 0) {
            rows_s[at[u]] = v[u].x;
            rows_s[at[u] + 1] = v[u].y;
          }
      }
    }
    sync();
    RTR(1);
    const int npairs = first_s[nrow];
    for (int p = tid; p < npairs; p += NT) {
      int r = 0;  // owning sample: last r with first_s[r] <= p
      for (int step = kResChunk; step > 0; step >>= 1)
        if (r + step < nrow && first_s[r + step] <= p) r += step;
      unsigned long long m = mask_s[r];
      for (int t = p - first_s[r]; t > 0; --t) m &= m - 1;  // the t-th candidate of r
      const int c = __ffsll(static_cast<long long>(m)) - 1;
      // padded stride d + 1: the lanes' rows / centroids fall in different banks
      const double* xr = rows_s + r * (d + 1);
      const double* mr = mu_s + c * (d + 1);
      double acc = 0.0;
#pragma unroll 8
      for (int j = 0; j < d; ++j) {   // the reference chain: sequential j, no FMA
        const double diff = __dsub_rn(xr[j], mr[j]);
        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
      }
      dist_s[p] = acc;
    }
    sync();
    RTR(2);
    for (int r = tid; r < nrow; r += NT) {
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
    sync();
    RTR(3);
    if (jj < d) {  // fold rows in list order; thread (rr, jj) owns cells (c, jj), c % R == rr
      for (int r = 0; r < nrow; ++r) {
        const int a = a_s[r];
        if (a % R == rr) {
          sums_s[a * d + jj] += rows_s[r * (d + 1) + jj];
          if (jj == 0) cnt_s[a] += 1;
        }
      }
    }
    RTR(4);
  }
  sync();
#ifdef DLX_KMEANS_TRACE
  if (tr && tid == 0)
    for (int i = 0; i < 5; ++i) tr[i] = tacc[i];
#endif
#undef RTR
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
  long long* part_counts;  // [grid][k]: per-CTA records (screened + re-checked samples)
  double* part_sums;       // [grid][k*d]
  long long* pend_idx;     // [grid][cap]
  unsigned long long* pend_mask;
  size_t used;
};

static ScreenedWs carve_screened(void* base, int64_t n, int d, int k, int grid) {
  const long long cap = pend_capacity(n, grid);
  Carve c(base);
  ScreenedWs w;
  w.pend_count = c.take<long long>(grid);
  const int parts = grid;
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
                         size_t ws_bytes, cudaStream_t stream, bool probe_only, double* mu_out) {
  DLX_REQUIRE(d >= 2 && d <= sk::kMaxD && (d & 1) == 0 && k >= 1 && k <= sk::kMaxK,
              DLX_ERR_GENERATION,
              "GenerationFailed: screened k-means needs even d <= %d and k <= %d (got d=%d k=%d)",
              sk::kMaxD, sk::kMaxK, d, k);
  DLX_REQUIRE((reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(mu) & 15) == 0,
              DLX_ERR_GENERATION, "GenerationFailed: screened k-means needs 16-byte aligned samples and centroids");
  // the fold accumulators hold <= 128*255 per tile in int32: at most 65,793 tiles per CTA
  DLX_REQUIRE(n <= (static_cast<int64_t>(60000) * sk::kTile) * sm_count(), DLX_ERR_GENERATION,
              "GenerationFailed: screened k-means takes at most %lld samples per launch",
              static_cast<long long>(60000) * sk::kTile * sm_count());
  if (probe_only) return DLX_OK;
  const int grid = screened_grid(n);
  const long long cap = pend_capacity(n, grid);
  ScreenedWs w = carve_screened(ws, n, d, k, grid);
  DLX_REQUIRE(ws && w.used <= ws_bytes, DLX_ERR_ARG, "k-means workspace too small (%zu < %zu)",
              ws_bytes, w.used);
  static const bool tracing = getenv("DLX_KMEANS_TRACE") != nullptr;
  long long* trace = nullptr;
  if (tracing) {
    DLX_CUDA(cudaMalloc(&trace, sizeof(long long) * grid * sk::kTraceTiles * 16));
    DLX_CUDA(cudaMemsetAsync(trace, 0, sizeof(long long) * grid * sk::kTraceTiles * 16, stream));
  }
  // 32-byte row loads when every lane's four columns are 32-byte aligned
  const bool wide = (d % 4 == 0) && (reinterpret_cast<uintptr_t>(x) % 32 == 0);
  auto kern = !wide ? sk::kmeans_screened_kernel<0, false>
                    : (d == 64 && n >= sk::kTile ? sk::kmeans_screened_kernel<64, true>
                                                 : sk::kmeans_screened_kernel<0, true>);
  DLX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sk::kSmemBytes)));
  DLX_CUDA(launch_pdl(kern, dim3(grid), dim3(sk::kThreads), sk::kSmemBytes, stream,
                      x, n, d, k, mu, assign, w.part_counts, w.part_sums, w.pend_idx, w.pend_mask,
                      w.pend_count, cap, trace));
  DLX_LAUNCHED("kmeans_screened_kernel");
  if (trace) {  // debug only: mean event offsets (cycles) relative to the converter's tile start
    std::vector<long long> h(static_cast<size_t>(grid) * sk::kTraceTiles * 16);
    DLX_CUDA(cudaStreamSynchronize(stream));
    DLX_CUDA(cudaMemcpy(h.data(), trace, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
    cudaFree(trace);
    const char* names[16] = {"screen_issued", "fold_issued", "conv_begin", "conv_got_buf", "conv_done",
                             "epi_begin", "epi_got_tfull", "epi_oh_done", "scr_got_afull", "scr_got_tempty",
                             "conv7_done", "epi_got_cfull", "epi_tmem_drained", "fold_got_oh",
                             "epi_pre_ohwait", "epi_post_ohwait"};
    double avg[16] = {0}, per_tile = 0;
    long cnt = 0;
    for (int b = 0; b < grid; ++b)
      for (int m = 8; m < sk::kTraceTiles - 2; ++m) {
        const long long* r = &h[(static_cast<size_t>(b) * sk::kTraceTiles + m) * 16];
        const long long* r1 = r + 16;
        if (r[2] == 0 || r1[2] == 0) continue;
        for (int e = 0; e < 16; ++e) avg[e] += static_cast<double>(r[e] - r[2]);
        per_tile += static_cast<double>(r1[2] - r[2]);
        ++cnt;
      }
    {
      double ph[6] = {0};
      for (int b = 0; b < grid; ++b) {
        const long long* r = &h[(static_cast<size_t>(b) * sk::kTraceTiles + sk::kTraceTiles - 1) * 16];
        for (int e = 0; e < 6; ++e) ph[e] += static_cast<double>(r[e] - r[0]) / grid;
      }
      fprintf(stderr, "[dlx phases] prologue %.0f; tiles done (fold_done) %+.0f; flush %+.0f; re-checks %+.0f; exit %+.0f cycles (mtiles %d)\n",
              ph[1], ph[2], ph[3], ph[4], ph[5], static_cast<int>((n + sk::kTile - 1) / sk::kTile / grid));
      double rt[5] = {0};
      for (int b = 0; b < grid; ++b)
        for (int e = 0; e < 5; ++e)
          rt[e] += static_cast<double>(h[(static_cast<size_t>(b) * sk::kTraceTiles + sk::kTraceTiles - 1) * 16 + 8 + e]) / grid;
      fprintf(stderr, "[dlx re-checks] list %.0f gather %.0f chains %.0f merge %.0f fold %.0f cycles\n",
              rt[0], rt[1], rt[2], rt[3], rt[4]);
    }
    if (cnt) {
      fprintf(stderr, "[dlx trace] tile period %.0f cycles;", per_tile / cnt);
      for (int e = 0; e < 16; ++e) fprintf(stderr, " %s %+.0f", names[e], avg[e] / cnt);
      fprintf(stderr, "\n");
    }
  }
  return kmeans_finalize(w.part_counts, w.part_sums, grid, k, d, counts, sums,
                         stream, mu_out);
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
