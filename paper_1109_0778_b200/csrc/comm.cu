// comm.cu — sample-sharded multi-GPU mode: one process per GPU, each rank runs
// the fused multiloop on its contiguous sample shard, then the partial activation records
// (k-means counts/sums, logreg gradient, GDA class sums / scatter, GroupBy counts) are
// summed across ranks with NCCL allReduce over NVLink / NVSwitch.  The unique id is
// exchanged by the caller (torch.distributed store / broadcast in the Python host layer).
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"

// NCCL is opened on first use (dlopen), not linked: a process that already loaded an NCCL
// (torch's bundled one) keeps using it, and libdlx.so never drags a second libnccl.so.2 into a
// process before torch's own.  Order: an NCCL already in the process, $DLX_NCCL_LIB, then the
// default search path.
namespace {
struct NcclApi {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  bool ok = false;
};
const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h && getenv("DLX_NCCL_LIB")) h = dlopen(getenv("DLX_NCCL_LIB"), RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define DLX_SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f))
    DLX_SYM(GetUniqueId);
    DLX_SYM(CommInitRank);
    DLX_SYM(CommDestroy);
    DLX_SYM(AllReduce);
    DLX_SYM(GroupStart);
    DLX_SYM(GroupEnd);
    DLX_SYM(GetErrorString);
#undef DLX_SYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce && api.GroupStart &&
             api.GroupEnd && api.GetErrorString;
  });
  return api;
}
}  // namespace

#define DLX_NCCL_API()                                                              \
  const NcclApi& N = nccl();                                                        \
  DLX_REQUIRE(N.ok, DLX_ERR_COMM, "NCCL unavailable: libnccl.so.2 could not be opened")

struct dlx_comm_s {
  ncclComm_t comm;
  int nranks;
  int rank;
};

static_assert(sizeof(ncclUniqueId) == DLX_COMM_ID_BYTES, "ncclUniqueId size");

#define DLX_NCCL(call)                                                         \
  do {                                                                         \
    ncclResult_t _r = (call);                                                  \
    if (_r != ncclSuccess) {                                                   \
      ::dlx::set_error("%s: %s", #call, N.GetErrorString(_r));                 \
      return DLX_ERR_COMM;                                                     \
    }                                                                          \
  } while (0)

extern "C" {

int dlx_comm_unique_id(uint8_t* h_id) {
  DLX_REQUIRE(h_id, DLX_ERR_ARG, "null id");
  DLX_NCCL_API();
  ncclUniqueId id;
  DLX_NCCL(N.GetUniqueId(&id));
  std::memcpy(h_id, &id, sizeof(id));
  return DLX_OK;
}

int dlx_comm_init(dlx_comm_t* comm, const uint8_t* h_id, int nranks, int rank) {
  DLX_REQUIRE(comm && h_id && nranks > 0 && rank >= 0 && rank < nranks, DLX_ERR_ARG,
              "comm init: bad args");
  DLX_NCCL_API();
  ncclUniqueId id;
  std::memcpy(&id, h_id, sizeof(id));
  auto* c = new dlx_comm_s{nullptr, nranks, rank};
  ncclResult_t r = N.CommInitRank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    dlx::set_error("ncclCommInitRank: %s", N.GetErrorString(r));
    return DLX_ERR_COMM;
  }
  *comm = c;
  return DLX_OK;
}

int dlx_comm_destroy(dlx_comm_t comm) {
  if (!comm) return DLX_OK;
  DLX_NCCL_API();
  ncclResult_t r = N.CommDestroy(comm->comm);
  delete comm;
  if (r != ncclSuccess) {
    dlx::set_error("ncclCommDestroy: %s", N.GetErrorString(r));
    return DLX_ERR_COMM;
  }
  return DLX_OK;
}

int dlx_comm_allreduce_sum(dlx_comm_t comm, void* d_buf, int64_t count, int dtype,
                           dlx_stream_t stream) {
  DLX_REQUIRE(comm && (d_buf || count == 0) && count >= 0, DLX_ERR_ARG, "allreduce: bad args");
  DLX_REQUIRE(dtype == 0 || dtype == 1, DLX_ERR_ARG, "allreduce: dtype must be 0 (f64) or 1 (i64)");
  if (count == 0) return DLX_OK;
  DLX_NCCL_API();
  DLX_NCCL(N.AllReduce(d_buf, d_buf, static_cast<size_t>(count),
                         dtype == 0 ? ncclFloat64 : ncclInt64, ncclSum, comm->comm, stream));
  return DLX_OK;
}

int dlx_comm_allreduce_sum_group(dlx_comm_t comm, void* const* d_bufs, const int64_t* counts,
                                 const int* dtypes, int nbufs, dlx_stream_t stream) {
  DLX_REQUIRE(comm && d_bufs && counts && dtypes && nbufs >= 0, DLX_ERR_ARG, "allreduce group: bad args");
  for (int i = 0; i < nbufs; ++i)
    DLX_REQUIRE((dtypes[i] == 0 || dtypes[i] == 1) && counts[i] >= 0 && (d_bufs[i] || counts[i] == 0),
                DLX_ERR_ARG, "allreduce group: bad buffer %d", i);
  DLX_NCCL_API();
  DLX_NCCL(N.GroupStart());
  for (int i = 0; i < nbufs; ++i) {
    if (counts[i] == 0) continue;
    const ncclResult_t r = N.AllReduce(d_bufs[i], d_bufs[i], static_cast<size_t>(counts[i]),
                                         dtypes[i] == 0 ? ncclFloat64 : ncclInt64, ncclSum,
                                         comm->comm, stream);
    if (r != ncclSuccess) {
      N.GroupEnd();
      dlx::set_error("ncclAllReduce: %s", N.GetErrorString(r));
      return DLX_ERR_COMM;
    }
  }
  DLX_NCCL(N.GroupEnd());
  return DLX_OK;
}

}  // extern "C"
