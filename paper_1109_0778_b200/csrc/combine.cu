// combine.cu — the combine step of the activation-record protocol (the
// runtime merges per-chunk records with combine(__act, rhs)).  Each multiloop kernel writes
// one partial record per CTA; this kernel folds them with a fixed shape (32 warps x strided
// partials, then an ordered 32-way sum), so results are deterministic for a given grid and
// the partial loads are coalesced and issued many at a time instead of as one sequential
// chain per output.
#include "common.cuh"

namespace dlx {

constexpr int kCombWarps = 32;   // warps per block: partial p goes to warp p % 32

template <class Tin, class Tout>
__device__ __forceinline__ void combine_columns(const Tin* __restrict__ parts, int nparts, long long width,
                                                Tout* __restrict__ out, long long block) {
  __shared__ Tout red[kCombWarps][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long e = block * 32 + lane;
  Tout a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  if (e < width) {
    int p = warp;
    // 16 loads in flight per lane, then the adds in the 4-accumulator order of the loop below
    // (a_u takes parts p + u*32, p + (u+4)*32, ...): one L2 round trip instead of four
    for (; p + 15 * kCombWarps < nparts; p += 16 * kCombWarps) {
      Tin v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = parts[static_cast<size_t>(p + u * kCombWarps) * width + e];
#pragma unroll
      for (int u = 0; u < 16; u += 4) {
        a0 += static_cast<Tout>(v[u]);
        a1 += static_cast<Tout>(v[u + 1]);
        a2 += static_cast<Tout>(v[u + 2]);
        a3 += static_cast<Tout>(v[u + 3]);
      }
    }
    for (; p + 3 * kCombWarps < nparts; p += 4 * kCombWarps) {
      a0 += static_cast<Tout>(parts[static_cast<size_t>(p) * width + e]);
      a1 += static_cast<Tout>(parts[static_cast<size_t>(p + kCombWarps) * width + e]);
      a2 += static_cast<Tout>(parts[static_cast<size_t>(p + 2 * kCombWarps) * width + e]);
      a3 += static_cast<Tout>(parts[static_cast<size_t>(p + 3 * kCombWarps) * width + e]);
    }
    for (; p < nparts; p += kCombWarps) a0 += static_cast<Tout>(parts[static_cast<size_t>(p) * width + e]);
  }
  red[warp][lane] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  if (warp == 0 && e < width) {
    Tout s = red[0][lane];
#pragma unroll
    for (int w = 1; w < kCombWarps; ++w) s += red[w][lane];
    out[e] = s;
  }
}

template <class Tin, class Tout>
__global__ void __launch_bounds__(kCombWarps * 32)
combine_partials_kernel(const Tin* __restrict__ parts, int nparts, long long width,
                        Tout* __restrict__ out, const int* __restrict__ skip) {
  pdl_wait();   // programmatic dependent launch: inputs are final from here on
  pdl_trigger();
  if (skip != nullptr && *skip) return;   // a device-side decision (GDA fit fallback)
  combine_columns<Tin, Tout>(parts, nparts, width, out, blockIdx.x);
}

// two records of one multiloop (e.g. k-means sums and counts) in one launch: the first
// blocks fold the fp64 record, the rest the int64 record
__global__ void __launch_bounds__(kCombWarps * 32)
combine_pair_kernel(const double* __restrict__ pf, long long wf, double* __restrict__ of,
                    const long long* __restrict__ pi, long long wi, long long* __restrict__ oi,
                    int nparts) {
  pdl_wait();   // the multiloop that wrote the partials has completed
  pdl_trigger();
  const long long bf = (wf + 31) / 32;
  if (blockIdx.x < bf) combine_columns<double, double>(pf, nparts, wf, of, blockIdx.x);
  else combine_columns<long long, long long>(pi, nparts, wi, oi, blockIdx.x - bf);
}

// The single-pass GDA fit's combine and finalize in one launch (gda_dmma.cu): the first blocks
// fold the CTAs' S' records, the next the shifted class sums, one block the class-1 counts —
// each as combine_columns does — and the last block to finish (a completion counter that the
// fit kernel zeroed and this block resets, so graph replays start from zero) computes
// mu_c = shift_c + sd_c / n_c, S = S' - sum_c sd_c sd_c^T / n_c and the certification flag
// (every diagonal correction <= 0.99 of S'_jj; also false for NaN / inf): the arithmetic of
// the former separate finalize kernel, with its inputs read from L2 (written by other blocks).
// (Folding the class sums redundantly in every block so each finalizes its own S columns
// measured slower: 18 vs 12 us, r315.)
__global__ void __launch_bounds__(kCombWarps * 32)
gda_fit_combine_kernel(const double* __restrict__ parts, const double* __restrict__ parts_sd,
                       const long long* __restrict__ parts_n1, int nparts, int d, double* __restrict__ Sp,
                       double* __restrict__ sd, long long* __restrict__ n1p, int64_t n,
                       const double* __restrict__ shift, unsigned* __restrict__ counter,
                       long long* __restrict__ n1_out, double* __restrict__ mu0, double* __restrict__ mu1,
                       double* __restrict__ S, int* __restrict__ ok, const double* __restrict__ parts_q,
                       double* __restrict__ qmax) {
  pdl_wait();
  pdl_trigger();
  const long long wS = static_cast<long long>(d) * d, bS = (wS + 31) / 32, bsd = (2LL * d + 31) / 32;
  if (blockIdx.x < bS) combine_columns<double, double>(parts, nparts, wS, Sp, blockIdx.x);
  else if (blockIdx.x < bS + bsd) combine_columns<double, double>(parts_sd, nparts, 2LL * d, sd, blockIdx.x - bS);
  else if (blockIdx.x == bS + bsd) combine_columns<long long, long long>(parts_n1, nparts, 1, n1p, 0);
  else {   // the int8 fit's quanta: max over the CTAs per column (inf marks an out-of-range CTA)
    __shared__ double qred[kCombWarps][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int j = static_cast<int>(blockIdx.x - bS - bsd - 1) * 32 + lane;
    double q = 0.0;
    if (j < d)
      for (int p = warp; p < nparts; p += kCombWarps) q = fmax(q, parts_q[static_cast<size_t>(p) * d + j]);
    qred[warp][lane] = q;
    __syncthreads();
    if (warp == 0 && j < d) {
      for (int w = 1; w < kCombWarps; ++w) q = fmax(q, qred[w][lane]);
      qmax[j] = q;
    }
  }
  __shared__ int last, bad;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
    bad = 0;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ double sd_s[128], sq_s[128];   // the class sums (d <= 64) and sums / n_c
  const long long n1 = __ldcg(n1p), n0 = n - n1;
  const double dn0 = static_cast<double>(n0), dn1 = static_cast<double>(n1);
  for (int e = threadIdx.x; e < 2 * d; e += blockDim.x) {
    sd_s[e] = __ldcg(sd + e);
    sq_s[e] = sd_s[e] / (e < d ? dn0 : dn1);   // one division per (class, column), not per entry
  }
  __syncthreads();
  auto corr = [&](int a, int b) {   // sum_c sd_c[a] sd_c[b] / n_c, the same value for (a, b), (b, a)
    const int lo = min(a, b), hi = max(a, b);
    double c = 0.0;
    if (n0 > 0) c += sd_s[lo] * sq_s[hi];
    if (n1 > 0) c += sd_s[d + lo] * sq_s[d + hi];
    return c;
  };
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    mu0[j] = __ldcg(shift + j) + sq_s[j];        // an empty class: 0 / 0 -> NaN, as the reference
    mu1[j] = __ldcg(shift + 64 + j) + sq_s[d + j];
    const double cj = corr(j, j), sj = __ldcg(Sp + j * d + j);
    if (!(cj <= 0.99 * sj)) bad = 1;
    // int8 fit: every CTA's quantum <= 2^-30 of the column's RMS deviation about the shift
    if (parts_q != nullptr) {
      const double q = __ldcg(qmax + j) * 1073741824.0;
      if (!(q * q * static_cast<double>(n) <= sj)) bad = 1;
    }
  }
  for (long long e = threadIdx.x; e < wS; e += blockDim.x)
    S[e] = __ldcg(Sp + e) - corr(static_cast<int>(e / d), static_cast<int>(e % d));
  __syncthreads();
  if (threadIdx.x == 0) {
    *ok = !bad;
    *n1_out = n1;
    *counter = 0u;
  }
}

int gda_fit_combine(const double* parts, const double* parts_sd, const long long* parts_n1, int nparts, int d,
                    double* Sp, double* sd, long long* n1p, int64_t n, const double* shift, unsigned* counter,
                    long long* n1_out, double* mu0, double* mu1, double* S, int* ok, cudaStream_t s,
                    const double* parts_q, double* qmax) {
  const long long blocks = (static_cast<long long>(d) * d + 31) / 32 + (2LL * d + 31) / 32 + 1 +
                           (parts_q != nullptr ? (d + 31) / 32 : 0);
  DLX_CUDA(launch_pdl(gda_fit_combine_kernel, dim3(static_cast<unsigned>(blocks)), dim3(kCombWarps * 32), 0, s,
                      parts, parts_sd, parts_n1, nparts, d, Sp, sd, n1p, n, shift, counter, n1_out, mu0, mu1, S, ok,
                      parts_q, qmax));
  DLX_LAUNCHED("gda_fit_combine_kernel");
  return DLX_OK;
}

template <class Tin, class Tout>
static int launch_combine(const Tin* parts, int nparts, long long width, Tout* out,
                          cudaStream_t stream, const int* skip = nullptr) {
  if (width <= 0) return DLX_OK;
  const long long blocks = (width + 31) / 32;
  DLX_CUDA(launch_pdl(combine_partials_kernel<Tin, Tout>, dim3(static_cast<unsigned>(blocks)), dim3(kCombWarps * 32), 0, stream,
      parts, nparts, width, out, skip));
  DLX_LAUNCHED("combine_partials_kernel");
  return DLX_OK;
}

int combine_f64(const double* parts, int nparts, long long width, double* out, cudaStream_t s) {
  return launch_combine<double, double>(parts, nparts, width, out, s);
}
int combine_f64_unless(const double* parts, int nparts, long long width, double* out,
                       const int* d_skip, cudaStream_t s) {
  return launch_combine<double, double>(parts, nparts, width, out, s, d_skip);
}
int combine_i64(const long long* parts, int nparts, long long width, long long* out,
                cudaStream_t s) {
  return launch_combine<long long, long long>(parts, nparts, width, out, s);
}
int combine_u32_i64(const unsigned* parts, int nparts, long long width, long long* out,
                    cudaStream_t s) {
  return launch_combine<unsigned, long long>(parts, nparts, width, out, s);
}
int combine_f64_i64(const double* pf, long long wf, double* of, const long long* pi, long long wi,
                    long long* oi, int nparts, cudaStream_t s) {
  const long long blocks = (wf + 31) / 32 + (wi + 31) / 32;
  if (blocks <= 0) return DLX_OK;
  DLX_CUDA(launch_pdl(combine_pair_kernel, dim3(static_cast<unsigned>(blocks)), dim3(kCombWarps * 32), 0, s,
                      pf, wf, of, pi, wi, oi, nparts));
  DLX_LAUNCHED("combine_pair_kernel");
  return DLX_OK;
}

// k-means at one rank: the combine of (sums, counts) fused with the centroid update
// mu[c*d+j] = sums[c*d+j] / (double)counts[c] (kmeans_update_kernel's arithmetic).  A sums
// block also folds the counts of its columns' centroids (integer sums: the same value the
// counts blocks write), so the update needs no second launch.
__global__ void __launch_bounds__(kCombWarps * 32)
combine_kmeans_update_kernel(const double* __restrict__ pf, double* __restrict__ of,
                             const long long* __restrict__ pi, long long* __restrict__ oi, int k, int d,
                             int nparts, double* __restrict__ mu) {
  pdl_wait();   // the multiloop that wrote the partials has completed (it also read mu)
  pdl_trigger();
  const long long wf = static_cast<long long>(k) * d;
  const long long bf = (wf + 31) / 32;
  if (blockIdx.x >= bf) {
    combine_columns<long long, long long>(pi, nparts, k, oi, blockIdx.x - bf);
    return;
  }
  __shared__ long long cnt_s[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long e = static_cast<long long>(blockIdx.x) * 32 + lane;
  const int c = e < wf ? static_cast<int>(e / d) : 0;
  long long a = 0;   // count of my column's centroid, folded per warp then across warps
#pragma unroll 8
  for (int p = warp; p < nparts; p += kCombWarps) a += pi[static_cast<size_t>(p) * k + c];
  __shared__ long long cred[kCombWarps][33];
  cred[warp][lane] = a;
  combine_columns<double, double>(pf, nparts, wf, of, blockIdx.x);   // ends with __syncthreads + warp 0 write
  if (warp == 0) {
    long long t = 0;
    for (int w = 0; w < kCombWarps; ++w) t += cred[w][lane];
    cnt_s[lane] = t;
  }
  __syncthreads();
  if (warp == 0 && e < wf) mu[e] = of[e] / static_cast<double>(cnt_s[lane]);  // IEEE: 0/0 -> NaN
}

int combine_kmeans_update(const double* pf, double* of, const long long* pi, long long* oi, int k, int d,
                          int nparts, double* mu, cudaStream_t s) {
  const long long blocks = (static_cast<long long>(k) * d + 31) / 32 + (k + 31) / 32;
  DLX_CUDA(launch_pdl(combine_kmeans_update_kernel, dim3(static_cast<unsigned>(blocks)), dim3(kCombWarps * 32), 0,
                      s, pf, of, pi, oi, k, d, nparts, mu));
  DLX_LAUNCHED("combine_kmeans_update_kernel");
  return DLX_OK;
}

}  // namespace dlx
