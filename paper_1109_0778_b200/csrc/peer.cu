// peer.cu — one-shot allreduce of a partial activation record over peer memory, fused with
// the update that consumes it (the "deterministic alternative": every rank folds
// the per-rank records in ascending rank order, the executeDEG ascending-chunk combine of
// SPEC.md:648/658 lifted to ranks, so all ranks hold bit-identical results independent of any
// reduction tree).
//
// Each rank owns one exchange buffer (cudaMalloc, exported with cudaIpcGetMemHandle and opened
// by every peer; over NVSwitch the peers' loads are NVLink reads, on one device they are local):
//
//   [0, 2048)      flags[256]  uint64  flag[b] = last epoch block b of this rank published
//   [2048, 2056)   epoch       uint64  calls completed by this rank (read only by this rank)
//   [2056, 2064)   done        uint32  blocks of the current call that finished (last one bumps epoch)
//   [4096, ...)    two record slots of (cap - 4096) / 2 bytes, used by alternate calls
//
// A record is `items` items of `ni` int64 values followed by `nf` fp64 values (k-means: k
// centroids x {count, d sums}; logreg: d gradient entries; GroupBy: K counts).  Block b owns a
// contiguous item range: it copies its items of the local record into slot (epoch & 1),
// publishes flag[b] = epoch with a system-scope release, waits until every peer's flag[b] has
// reached the epoch, folds the peers' items rank 0, 1, ..., n-1 and writes the sum back over
// the local record, then applies the epilogue (k-means mu = sum / toDouble(count); BGD
// theta -= alpha * g).  Slot reuse is safe without a second barrier: a rank writes slot e&1
// again only at epoch e+2, after its call e+1 saw every peer publish e+1, and a peer publishes
// e+1 only after its call e, the last reader of that slot, has completed.
//
// This replaces {NCCL allReduce, update kernel} with one launch.  Polling has a 30 s limit and
// traps, so a missing peer fails loudly instead of hanging the device.
#include <algorithm>
#include <cstring>

#include "common.cuh"

namespace dlx {

constexpr int kPeerMaxRanks = 16;
constexpr int kPeerMaxBlocks = 256;
constexpr int kPeerThreads = 256;
constexpr int64_t kPeerHeader = 4096;

struct PeerArgs {
  char* bufs[kPeerMaxRanks];   // every rank's exchange buffer, mapped in this process
  int nranks, rank;
  int64_t slot_bytes;
  int64_t items;
  int ni, nf;
  int64_t items_per_block;
  long long* counts;           // local record in / global record out: items x ni
  double* sums;                // items x nf
  int epilogue;                // 0 none, 1 k-means update, 2 theta -= alpha * g
  double* out;
  double alpha;
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(kPeerThreads) peer_allreduce_kernel(const PeerArgs a) {
  pdl_wait();   // the local record (combine of this rank's per-CTA partials) is final
  pdl_trigger();
  __shared__ unsigned long long s_epoch;
  char* const mine = a.bufs[a.rank];
  auto* const flags = reinterpret_cast<unsigned long long*>(mine);
  auto* const epoch_p = reinterpret_cast<volatile unsigned long long*>(mine + 2048);
  auto* const done_p = reinterpret_cast<unsigned*>(mine + 2056);
  if (threadIdx.x == 0) s_epoch = *epoch_p + 1;
  __syncthreads();
  const unsigned long long e = s_epoch;
  const int64_t slot_off = kPeerHeader + static_cast<int64_t>(e & 1) * a.slot_bytes;
  const int rec = a.ni + a.nf;                        // 8-byte values per item
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * a.items_per_block;
  const int64_t i1 = min(a.items, i0 + a.items_per_block);
  const int64_t nv = (i1 - i0) * rec;                 // values this block owns

  // 1. publish this rank's items of the record into its slot
  auto* const myslot = reinterpret_cast<unsigned long long*>(mine + slot_off);
  for (int64_t v = threadIdx.x; v < nv; v += kPeerThreads) {
    const int64_t it = i0 + v / rec;
    const int f = static_cast<int>(v % rec);
    myslot[i0 * rec + v] = f < a.ni ? static_cast<unsigned long long>(a.counts[it * a.ni + f])
                                    : __double_as_longlong(a.sums[it * a.nf + (f - a.ni)]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    st_release_sys(flags + blockIdx.x, e);
  }
  // 2. wait for every peer's block b to publish the same epoch
  if (threadIdx.x < a.nranks && threadIdx.x != a.rank) {
    const auto* f = reinterpret_cast<const unsigned long long*>(a.bufs[threadIdx.x]) + blockIdx.x;
    const unsigned long long t0 = globaltimer();
    while (ld_acquire_sys(f) < e) {
      if (globaltimer() - t0 > 30ull * 1000000000ull) {
        printf("dlx peer_allreduce: rank %d block %d timed out waiting for rank %d (epoch %llu)\n",
               a.rank, blockIdx.x, threadIdx.x, e);
        __trap();
      }
      __nanosleep(200);
    }
  }
  __syncthreads();
  // 3. ordered fold over ranks, written over the local record, then the epilogue
  for (int64_t v = threadIdx.x; v < nv; v += kPeerThreads) {
    const int64_t it = i0 + v / rec;
    const int f = static_cast<int>(v % rec);
    const int64_t off = slot_off + (i0 * rec + v) * 8;
    if (f < a.ni) {
      long long s = 0;
      for (int q = 0; q < a.nranks; ++q)
        s += static_cast<long long>(__ldcv(reinterpret_cast<const unsigned long long*>(a.bufs[q] + off)));
      a.counts[it * a.ni + f] = s;
    } else {
      double s = __longlong_as_double(static_cast<long long>(
          __ldcv(reinterpret_cast<const unsigned long long*>(a.bufs[0] + off))));
      for (int q = 1; q < a.nranks; ++q)
        s = __dadd_rn(s, __longlong_as_double(static_cast<long long>(
                             __ldcv(reinterpret_cast<const unsigned long long*>(a.bufs[q] + off)))));
      a.sums[it * a.nf + (f - a.ni)] = s;
      if (a.epilogue == 2) {
        const int64_t j = it * a.nf + (f - a.ni);
        a.out[j] = __dsub_rn(a.out[j], __dmul_rn(a.alpha, s));
      }
    }
  }
  if (a.epilogue == 1) {   // k-means: mu[c][j] = sums[c][j] / toDouble(counts[c]) (0/0 -> NaN)
    __syncthreads();
    for (int64_t v = threadIdx.x; v < (i1 - i0) * a.nf; v += kPeerThreads) {
      const int64_t c = i0 + v / a.nf;
      const int64_t j = c * a.nf + v % a.nf;
      a.out[j] = a.sums[j] / static_cast<double>(a.counts[c * a.ni]);
    }
  }
  // 4. the last block to finish advances this rank's epoch for the next call
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(done_p, 1u) == gridDim.x - 1) {
      *done_p = 0;
      *epoch_p = e;
      __threadfence();
    }
  }
}

}  // namespace dlx

extern "C" {

int dlx_peer_alloc(int64_t bytes, void** d_ptr, uint8_t* h_handle) {
  DLX_REQUIRE(d_ptr && h_handle && bytes > dlx::kPeerHeader, DLX_ERR_ARG, "peer alloc: bad args");
  void* p = nullptr;
  DLX_CUDA(cudaMalloc(&p, static_cast<size_t>(bytes)));
  cudaError_t err = cudaMemset(p, 0, static_cast<size_t>(bytes));
  cudaIpcMemHandle_t h;
  if (err == cudaSuccess) err = cudaIpcGetMemHandle(&h, p);
  if (err != cudaSuccess) {
    cudaFree(p);
    return dlx::cuda_fail(err, "peer alloc");
  }
  static_assert(sizeof(cudaIpcMemHandle_t) == DLX_PEER_HANDLE_BYTES, "ipc handle size");
  memcpy(h_handle, &h, sizeof(h));
  *d_ptr = p;
  return DLX_OK;
}

int dlx_peer_open(const uint8_t* h_handle, void** d_ptr) {
  DLX_REQUIRE(d_ptr && h_handle, DLX_ERR_ARG, "peer open: bad args");
  cudaIpcMemHandle_t h;
  memcpy(&h, h_handle, sizeof(h));
  DLX_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return DLX_OK;
}

int dlx_peer_close(void* d_ptr) {
  if (d_ptr) DLX_CUDA(cudaIpcCloseMemHandle(d_ptr));
  return DLX_OK;
}

int dlx_peer_free(void* d_ptr) {
  if (d_ptr) DLX_CUDA(cudaFree(d_ptr));
  return DLX_OK;
}

int dlx_peer_allreduce(void* const* h_bufs, int nranks, int rank, int64_t cap_bytes, int64_t items,
                       int ni, int nf, int64_t* d_counts, double* d_sums, int epilogue,
                       double* d_out, double alpha, dlx_stream_t stream) {
  using namespace dlx;
  DLX_REQUIRE(h_bufs && nranks >= 1 && nranks <= kPeerMaxRanks && rank >= 0 && rank < nranks,
              DLX_ERR_ARG, "peer allreduce: bad ranks (%d of %d, max %d)", rank, nranks, kPeerMaxRanks);
  DLX_REQUIRE(items >= 0 && ni >= 0 && nf >= 0 && ni + nf > 0, DLX_ERR_ARG, "peer allreduce: bad record");
  DLX_REQUIRE((ni == 0 || d_counts) && (nf == 0 || d_sums), DLX_ERR_ARG, "peer allreduce: null record");
  DLX_REQUIRE(epilogue >= 0 && epilogue <= 2, DLX_ERR_ARG, "peer allreduce: bad epilogue");
  DLX_REQUIRE(epilogue == 0 || (d_out && nf > 0), DLX_ERR_ARG, "peer allreduce: epilogue needs out");
  DLX_REQUIRE(epilogue != 1 || ni == 1, DLX_ERR_ARG, "peer allreduce: k-means epilogue needs one count per item");
  PeerArgs a{};
  a.slot_bytes = (cap_bytes - kPeerHeader) / 2 / 8 * 8;
  DLX_REQUIRE(items * (ni + nf) * 8 <= a.slot_bytes, DLX_ERR_ARG,
              "peer allreduce: record of %lld bytes exceeds the %lld-byte slot",
              static_cast<long long>(items * (ni + nf) * 8), static_cast<long long>(a.slot_bytes));
  if (items == 0) return DLX_OK;
  for (int q = 0; q < nranks; ++q) {
    DLX_REQUIRE(h_bufs[q], DLX_ERR_ARG, "peer allreduce: null buffer for rank %d", q);
    a.bufs[q] = static_cast<char*>(h_bufs[q]);
  }
  a.nranks = nranks;
  a.rank = rank;
  a.items = items;
  a.ni = ni;
  a.nf = nf;
  // enough blocks that each moves a few KB; at most kPeerMaxBlocks flags
  const int64_t per_item = (ni + nf) * 8;
  int64_t blocks = std::min<int64_t>(kPeerMaxBlocks, std::max<int64_t>(1, items * per_item / 4096));
  a.items_per_block = (items + blocks - 1) / blocks;
  blocks = (items + a.items_per_block - 1) / a.items_per_block;
  a.counts = reinterpret_cast<long long*>(d_counts);
  a.sums = d_sums;
  a.epilogue = epilogue;
  a.out = d_out;
  a.alpha = alpha;
  DLX_CUDA(launch_pdl(peer_allreduce_kernel, dim3(static_cast<unsigned>(blocks)), dim3(kPeerThreads), 0,
                      static_cast<cudaStream_t>(stream), a));
  DLX_LAUNCHED("peer_allreduce_kernel");
  return DLX_OK;
}

}  // extern "C"
