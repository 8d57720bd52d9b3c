// kmeans_screened.cu — tcgen05 screened k-means (placeholder until the kernel lands).
#include "common.cuh"

namespace dlx {

size_t kmeans_screened_workspace_bytes(int64_t, int, int) { return 0; }

int kmeans_screened_step(const double*, int64_t, int, int, const double*, int32_t*, long long*,
                         double*, void*, size_t, cudaStream_t, bool) {
  set_error("GenerationFailed: screened k-means not built");
  return DLX_ERR_GENERATION;
}

}  // namespace dlx

extern "C" int dlx_kmeans_last_recheck_count(const void*, int64_t* h_count, dlx_stream_t) {
  if (h_count) *h_count = -1;
  return DLX_OK;
}
