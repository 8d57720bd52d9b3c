// groupby.cu — GroupBy / bucket-count multiloop.
//
// Reference formulation: nbuckets predicated count reduces `if (key(i) == b) cnt_b += 1`
// over one index traversal (count_where, proj/src/vectordsl.cpp:138-151), O(N*K) guards.
// Device plan: one pass over the keys with 128-bit loads; shared-memory privatised
// counters (several sub-histograms per CTA, one per warp group, to spread same-bucket
// contention), merged per CTA into uint32 partials and combined across CTAs in ascending
// order.  Buckets too many for shared memory use 64-bit global reductions.  Integer
// arithmetic, so results are exact and independent of the reduction order.
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"

namespace dlx {

constexpr int kGbThreads = 512;
constexpr size_t kGbSmemBudget = 96 * 1024;
constexpr int kGbPairThreads = 1024;               // two-CTA cluster path (groupby_pair_kernel)

constexpr size_t kGbPairSmemBudget = 200 * 1024;   // histogram slice per CTA
#ifndef DLX_GB_MAX_CLUSTER
#define DLX_GB_MAX_CLUSTER 4
#endif

struct GroupbyPlan {
  bool shared;   // shared-memory privatised path
  bool pair;     // CTA cluster, one histogram sliced across the cluster's shared memories
  int csize;     // cluster size (2, 4, 8)
  int copies;    // sub-histograms per CTA
  int grid;
  size_t smem;
};

static GroupbyPlan groupby_plan(int64_t n, int64_t nb) {
  GroupbyPlan p{};
  const size_t one = static_cast<size_t>(nb) * sizeof(unsigned);
  p.shared = one <= kGbSmemBudget;
  int per_sm = 2;
  if (p.shared) {
    p.copies = static_cast<int>(std::min<size_t>(kGbThreads / 32, kGbSmemBudget / one));
    p.copies = std::max(1, p.copies);
    // power of two so warp -> copy is a mask
    int c = 1;
    while (c * 2 <= p.copies) c *= 2;
    p.copies = c;
    p.smem = one * p.copies;
  } else {
    p.copies = 0;
    p.smem = 0;
    per_sm = 4;
    for (int c = 2; c <= DLX_GB_MAX_CLUSTER; c *= 2) {
      const size_t slice = static_cast<size_t>((nb + c - 1) / c) * sizeof(unsigned);
      if (slice <= kGbPairSmemBudget) {
        p.pair = true;
        p.csize = c;
        p.smem = slice;
        p.grid = (sm_count() / c) * c;   // one CTA per SM, whole clusters
        return p;
      }
    }
  }
  int64_t grid = static_cast<int64_t>(sm_count()) * per_sm;
  const int64_t need = (n / 2 + kGbThreads - 1) / kGbThreads;
  grid = std::max<int64_t>(1, std::min(grid, need));
  p.grid = static_cast<int>(grid);
  return p;
}

__device__ __forceinline__ void count_key(unsigned* h, long long key, long long nb) {
  if (static_cast<unsigned long long>(key) < static_cast<unsigned long long>(nb))
    atomicAdd(h + key, 1u);
}

__global__ void __launch_bounds__(kGbThreads)
groupby_smem_kernel(const long long* __restrict__ keys, int64_t n, long long nb, int copies,
                    unsigned* __restrict__ partials) {
  pdl_wait();   // programmatic dependent launch: inputs are final from here on
  pdl_trigger();
  extern __shared__ unsigned hist[];
  const int tid = threadIdx.x;
  const int total = static_cast<int>(nb) * copies;
  for (int e = tid; e < total; e += kGbThreads) hist[e] = 0;
  __syncthreads();
  unsigned* h = hist + static_cast<size_t>((tid >> 5) & (copies - 1)) * nb;

  // pairs of keys via 128-bit loads; 4 pairs in flight per thread
  const int64_t npairs = n >> 1;
  const longlong2* kp = reinterpret_cast<const longlong2*>(keys);
  const int64_t T = static_cast<int64_t>(gridDim.x) * kGbThreads;
  int64_t q = static_cast<int64_t>(blockIdx.x) * kGbThreads + tid;
  for (; q + 3 * T < npairs; q += 4 * T) {
    longlong2 v0 = __ldg(kp + q), v1 = __ldg(kp + q + T), v2 = __ldg(kp + q + 2 * T),
              v3 = __ldg(kp + q + 3 * T);
    count_key(h, v0.x, nb); count_key(h, v0.y, nb);
    count_key(h, v1.x, nb); count_key(h, v1.y, nb);
    count_key(h, v2.x, nb); count_key(h, v2.y, nb);
    count_key(h, v3.x, nb); count_key(h, v3.y, nb);
  }
  for (; q < npairs; q += T) {
    longlong2 v = __ldg(kp + q);
    count_key(h, v.x, nb);
    count_key(h, v.y, nb);
  }
  if ((n & 1) && blockIdx.x == 0 && tid == 0) count_key(h, keys[n - 1], nb);
  __syncthreads();
  unsigned* out = partials + static_cast<size_t>(blockIdx.x) * nb;
  for (long long b = tid; b < nb; b += kGbThreads) {
    unsigned acc = 0;
    for (int c = 0; c < copies; ++c) acc += hist[static_cast<size_t>(c) * nb + b];
    out[b] = acc;
  }
}

// Buckets past one CTA's shared memory (24K < K <= 100K, e.g. the K = 65,536 point of the
// SURVEY §8 a7 sweep): a thread-block cluster of two CTAs (two SMs) splits ONE u32 histogram
// between its shared memories.  Both CTAs stream the cluster's keys in lockstep and each
// counts the keys of its own half with shared-memory atomics; the cluster co-schedules the
// pair, so the partner's read of every line is an L2 hit and HBM sees each key once (r86:
// 8.0 GB read for 1e9 keys).  Measured against the alternative of one read per key with the
// foreign half incremented remotely through distributed shared memory: 1.61 ms vs 5.42 ms at
// 1e9 keys, K = 65,536 (remote DSMEM atomics are the bottleneck); the global-atomics path
// this replaces took 6.54 ms.
// Cluster size kC = 2 or 4 (DLX_GB_MAX_CLUSTER; 8 is built but loses to global atomics, r89):
// each CTA holds a 1/kC slice of the histogram and every key of the cluster's stream is read
// by kC SMs (L2 hits after the first), so the L2->SM stream grows with kC.
template <int kC>
__global__ void __cluster_dims__(kC, 1, 1) __launch_bounds__(kGbPairThreads, 1)
groupby_pair_kernel(const long long* __restrict__ keys, int64_t n, long long nb,
                    unsigned* __restrict__ partials) {
  namespace cg = cooperative_groups;
  extern __shared__ unsigned hist[];
  const long long per = (nb + kC - 1) / kC;
  const unsigned rank = cg::this_cluster().block_rank();
  for (long long e = threadIdx.x; e < per; e += kGbPairThreads) hist[e] = 0;
  __syncthreads();
  pdl_wait();  // programmatic dependent launch: keys are final from here on
  pdl_trigger();
  const long long lo = std::min<long long>(nb, rank * per), w = std::min<long long>(per, nb - lo);
  const unsigned long long lo_k = static_cast<unsigned long long>(lo), w_k = static_cast<unsigned long long>(w);
  auto count = [&](long long key) {
    const unsigned long long rel = static_cast<unsigned long long>(key) - lo_k;   // < 0 wraps
    if (rel < w_k) atomicAdd(hist + rel, 1u);
  };
  const int64_t npairs = n >> 1;
  const longlong2* kp = reinterpret_cast<const longlong2*>(keys);
  const int64_t T = static_cast<int64_t>(gridDim.x / kC) * kGbPairThreads;
  int64_t q = static_cast<int64_t>(blockIdx.x / kC) * kGbPairThreads + threadIdx.x;
  for (; q + 3 * T < npairs; q += 4 * T) {
    longlong2 v0 = __ldg(kp + q), v1 = __ldg(kp + q + T), v2 = __ldg(kp + q + 2 * T),
              v3 = __ldg(kp + q + 3 * T);
    count(v0.x); count(v0.y); count(v1.x); count(v1.y);
    count(v2.x); count(v2.y); count(v3.x); count(v3.y);
  }
  for (; q < npairs; q += T) {
    longlong2 v = __ldg(kp + q);
    count(v.x);
    count(v.y);
  }
  if ((n & 1) && blockIdx.x / kC == 0 && threadIdx.x == 0) count(keys[n - 1]);   // every slice looks
  __syncthreads();
  unsigned* out = partials + static_cast<size_t>(blockIdx.x / kC) * nb + lo;
  for (long long b = threadIdx.x; b < w; b += kGbPairThreads) out[b] = hist[b];
}

__global__ void __launch_bounds__(kGbThreads)
groupby_global_kernel(const long long* __restrict__ keys, int64_t n, long long nb,
                      unsigned long long* __restrict__ counts) {
  pdl_wait();   // programmatic dependent launch: inputs are final from here on
  pdl_trigger();
  const int64_t T = static_cast<int64_t>(gridDim.x) * kGbThreads;
  const int64_t npairs = n >> 1;
  const longlong2* kp = reinterpret_cast<const longlong2*>(keys);
  for (int64_t q = static_cast<int64_t>(blockIdx.x) * kGbThreads + threadIdx.x; q < npairs;
       q += T) {
    longlong2 v = __ldg(kp + q);
    if (static_cast<unsigned long long>(v.x) < static_cast<unsigned long long>(nb))
      atomicAdd(counts + v.x, 1ull);
    if (static_cast<unsigned long long>(v.y) < static_cast<unsigned long long>(nb))
      atomicAdd(counts + v.y, 1ull);
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    long long key = keys[n - 1];
    if (static_cast<unsigned long long>(key) < static_cast<unsigned long long>(nb))
      atomicAdd(counts + key, 1ull);
  }
}

}  // namespace dlx

using namespace dlx;

extern "C" {

size_t dlx_groupby_workspace_bytes(int64_t n, int64_t nbuckets) {
  GroupbyPlan p = groupby_plan(n, nbuckets);
  if (p.pair) return static_cast<size_t>(p.grid / p.csize) * nbuckets * sizeof(unsigned) + 256;
  if (!p.shared) return 256;
  return static_cast<size_t>(p.grid) * nbuckets * sizeof(unsigned) + 256;
}

int dlx_groupby_count(const int64_t* d_keys, int64_t n, int64_t nbuckets, int64_t* d_counts,
                      void* d_workspace, size_t workspace_bytes, dlx_stream_t stream) {
  DLX_REQUIRE(n >= 0 && nbuckets > 0, DLX_ERR_ARG, "groupby: bad shape");
  DLX_REQUIRE(d_counts && (d_keys || n == 0), DLX_ERR_ARG, "groupby: null buffer");
  DLX_REQUIRE((reinterpret_cast<uintptr_t>(d_keys) & 15) == 0, DLX_ERR_ARG,
              "groupby: keys must be 16-byte aligned");
  GroupbyPlan p = groupby_plan(n, nbuckets);
  if (p.pair) {
    const int clusters = p.grid / p.csize;
    const size_t need = static_cast<size_t>(clusters) * nbuckets * sizeof(unsigned);
    DLX_REQUIRE(d_workspace && workspace_bytes >= need, DLX_ERR_ARG,
                "groupby: workspace too small (%zu < %zu)", workspace_bytes, need);
    unsigned* partials = static_cast<unsigned*>(d_workspace);
    auto kern = p.csize == 2 ? groupby_pair_kernel<2> : p.csize == 4 ? groupby_pair_kernel<4> : groupby_pair_kernel<8>;
    DLX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem)));
    DLX_CUDA(launch_pdl(kern, dim3(p.grid), dim3(kGbPairThreads), p.smem, stream,
                        reinterpret_cast<const long long*>(d_keys), n, nbuckets, partials));
    DLX_LAUNCHED("groupby_pair_kernel");
    return combine_u32_i64(partials, clusters, nbuckets, reinterpret_cast<long long*>(d_counts), stream);
  }
  if (!p.shared) {
    DLX_CUDA(cudaMemsetAsync(d_counts, 0, sizeof(int64_t) * nbuckets, stream));
    if (n == 0) return DLX_OK;
    DLX_CUDA(launch_pdl(groupby_global_kernel, dim3(p.grid), dim3(kGbThreads), 0, stream, 
        reinterpret_cast<const long long*>(d_keys), n, nbuckets,
        reinterpret_cast<unsigned long long*>(d_counts)));
    DLX_LAUNCHED("groupby_global_kernel");
    return DLX_OK;
  }
  const size_t need = static_cast<size_t>(p.grid) * nbuckets * sizeof(unsigned);
  DLX_REQUIRE(d_workspace && workspace_bytes >= need, DLX_ERR_ARG,
              "groupby: workspace too small (%zu < %zu)", workspace_bytes, need);
  unsigned* partials = static_cast<unsigned*>(d_workspace);
  DLX_CUDA(cudaFuncSetAttribute(groupby_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(p.smem)));
  DLX_CUDA(launch_pdl(groupby_smem_kernel, dim3(p.grid), dim3(kGbThreads), p.smem, stream, 
      reinterpret_cast<const long long*>(d_keys), n, nbuckets, p.copies, partials));
  DLX_LAUNCHED("groupby_smem_kernel");
  return combine_u32_i64(partials, p.grid, nbuckets, reinterpret_cast<long long*>(d_counts), stream);
}

}  // extern "C"
