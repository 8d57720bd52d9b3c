/*
 * dlx.h — C ABI of the B200 fused-multiloop executor ("dlx": Delite loop executor).
 *
 * This is the drop-in boundary for the reference's missing parallel executor.  The
 * reference (stagekit, /root/reference/proj) lowers each fused multiloop
 * (LoopPayload, proj/include/stagekit/node.hpp:60-81) to sequential MiniC text in
 * emit_parallel_loop (proj/src/codegen.cpp:345-433) and declares, but never implements,
 *     RunResult interpret(const minic::Program&, uint64_t seed)   (interp.hpp:10)
 * and specifies, in prose only, executeDEG / scheduleDEG.  Each entry
 * point below replaces the execution of one recognised multiloop family; the C++ host
 * executor (include/dlx/executor.hpp) maps LoopPayload-shaped descriptors onto them.
 *
 * Conventions (all entry points):
 *   - plain pointers and sizes only; device pointers are marked `d_`, host pointers `h_`;
 *   - the caller owns every buffer and the stream; launchers never allocate (scratch comes
 *     from a caller-provided workspace sized by the matching *_workspace_bytes query);
 *   - return DLX_OK (0) or an error code; dlx_last_error() returns the thread-local message;
 *   - no exceptions cross this boundary;
 *   - reference element types: Int = int64, Double = fp64 (types.hpp:11-20).  Collect
 *     outputs that hold centroid indices are int32 on the device (k < 2^31) and are widened
 *     to Int by the host layer on download.
 */
#ifndef DLX_H_
#define DLX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* dlx_stream_t; /* == cudaStream_t; NULL = legacy default stream */

/* Status codes.  DLX_ERR_GENERATION mirrors StagingError::GenerationFailed
 * (errors.hpp:19, raised by codegen.cpp:66-71 for loops no emitter handles);
 * DLX_ERR_TRAP mirrors TrapError (errors.hpp:46-67, CLI exit 3). */
enum {
  DLX_OK = 0,
  DLX_ERR_CUDA = 1,       /* CUDA runtime / driver failure */
  DLX_ERR_GENERATION = 2, /* shape or family this executor cannot lower (no CPU fallback) */
  DLX_ERR_TRAP = 3,       /* runtime trap (division by zero, index out of bounds) */
  DLX_ERR_ARG = 4,        /* invalid argument (null pointer, negative size) */
  DLX_ERR_COMM = 5        /* NCCL failure */
};

const char* dlx_last_error(void);
const char* dlx_version(void);
/* kernels this library has launched since it was loaded (all devices, all threads) */
uint64_t dlx_launch_count(void);

/* ---- device / memory (device mirrors of VecData, runtime.hpp:44-72) ------------------ */
int dlx_device_count(int* count);
int dlx_set_device(int device);
int dlx_sm_count(int* sms);
int dlx_malloc(void** d_ptr, size_t bytes);
int dlx_free(void* d_ptr);
int dlx_host_alloc(void** h_ptr, size_t bytes); /* pinned, for staged upload/download */
int dlx_host_free(void* h_ptr);
int dlx_memcpy_h2d(void* d_dst, const void* h_src, size_t bytes, dlx_stream_t stream);
int dlx_memcpy_d2h(void* h_dst, const void* d_src, size_t bytes, dlx_stream_t stream);
int dlx_memset(void* d_dst, int value, size_t bytes, dlx_stream_t stream);
int dlx_stream_create(dlx_stream_t* stream);
int dlx_stream_destroy(dlx_stream_t stream);
int dlx_stream_sync(dlx_stream_t stream);

/* ---- synthetic sources: VectorRand / VectorRandInt with the reference Rng ------------ */
/* Rng (runtime.hpp:86-96): state = state*6364136223846793005 + 1442695040888963407;
 * next_unit = (state>>11)*2^-53; next_int(b) = (int64)(next_unit*b).  Element t of the
 * output is draw number first_draw + t of Rng(seed) (0-based), computed on the device by
 * affine skip-ahead, so device data is bit-identical to drawing sequentially on the host. */
int dlx_rng_units(double* d_out, int64_t n, uint64_t seed, uint64_t first_draw,
                  dlx_stream_t stream);
int dlx_rng_ints(int64_t* d_out, int64_t n, int64_t bound, uint64_t seed, uint64_t first_draw,
                 dlx_stream_t stream);

/* ---- k-means iteration: one fused multiloop = 1 collect (argmin) + k*(d+1) predicated
 *      reduces (counts, per-centroid sums), SURVEY §8 a4 ---------------------------------- */
/* x: n*d row-major fp64; mu: k*d fp64.  Writes d_assign[n] (int32, optional: may be NULL),
 * d_counts[k] (int64) and d_sums[k*d] (fp64) for this shard.  Assignments are bit-exact
 * with the reference argmin chain (sequential j-order (x-mu)^2 fp64 sums without FMA,
 * strict <, chain start 1e300 / index 0).  method: DLX_KMEANS_AUTO picks the tcgen05
 * screened kernel when the shape allows it, else the direct fp64 kernel. */
enum { DLX_KMEANS_AUTO = 0, DLX_KMEANS_DIRECT = 1, DLX_KMEANS_SCREENED = 2 };
size_t dlx_kmeans_workspace_bytes(int64_t n, int32_t d, int32_t k);
int dlx_kmeans_step(const double* d_x, int64_t n, int32_t d, int32_t k, const double* d_mu,
                    int32_t* d_assign, int64_t* d_counts, double* d_sums, void* d_workspace,
                    size_t workspace_bytes, int method, dlx_stream_t stream);
/* One whole k-means iteration at one rank: dlx_kmeans_step, then d_mu updated in place with
 * dlx_kmeans_update's arithmetic, the update fused into the step's combine launch (one launch
 * fewer per iteration).  Results bit-identical to step + update.  Replaces the reference's
 * staged iteration: fused loop + k*d `mu.update(c*d+j, sum/toDouble(count))` (vectordsl.cpp:90-103). */
int dlx_kmeans_iteration(const double* d_x, int64_t n, int32_t d, int32_t k, double* d_mu,
                         int32_t* d_assign, int64_t* d_counts, double* d_sums, void* d_workspace,
                         size_t workspace_bytes, int method, dlx_stream_t stream);
/* mu[c*d+j] = sums[c*d+j] / (double)counts[c]  (empty cluster -> 0/0 = NaN) */
int dlx_kmeans_update(const int64_t* d_counts, const double* d_sums, int32_t k, int32_t d,
                      double* d_mu, dlx_stream_t stream);
/* Number of samples the last screened step on this workspace (same n, d, k) re-evaluated
 * with the exact reference chain (diagnostic; synchronises the stream). */
int dlx_kmeans_last_recheck_count(const void* d_workspace, int64_t n, int32_t d, int32_t k,
                                  int64_t* h_count, dlx_stream_t stream);

/* ---- GroupBy / bucket-reduce: counts[b] = #{i : keys[i] == b}, b in [0, nbuckets) ------ */
/* (the reference expresses this as nbuckets predicated count reduces).
 * keys outside [0, nbuckets) are not counted.  Exact int64. */
size_t dlx_groupby_workspace_bytes(int64_t n, int64_t nbuckets);
int dlx_groupby_count(const int64_t* d_keys, int64_t n, int64_t nbuckets, int64_t* d_counts,
                      void* d_workspace, size_t workspace_bytes, dlx_stream_t stream);

/* ---- logistic regression gradient: fused dot -> sigmoid -> d reduces ----- */
/* grad_j = sum_i (1/(1+exp(-theta.x_i)) - y_i) * x_ij.  exp is a documented extension
 * (the reference op set, node.hpp:15-27, has none). */
size_t dlx_logreg_workspace_bytes(int64_t n, int32_t d);
int dlx_logreg_grad(const double* d_x, const int64_t* d_y, int64_t n, int32_t d,
                    const double* d_theta, double* d_grad, void* d_workspace,
                    size_t workspace_bytes, dlx_stream_t stream);
/* fp32 storage opt-in (the reference Ty has no fp32, types.hpp:11-20): x held
 * as float (half the bytes of the HBM-bound stream), every element promoted exactly to double,
 * the arithmetic that of dlx_logreg_grad — so the gradient is bit-identical to dlx_logreg_grad
 * on the promoted matrix.  Same workspace as dlx_logreg_grad. */
int dlx_logreg_grad_f32(const float* d_x, const int64_t* d_y, int64_t n, int32_t d,
                        const double* d_theta, double* d_grad, void* d_workspace,
                        size_t workspace_bytes, dlx_stream_t stream);
/* The staged logistic-regression loop (the collect form the reference fuses into
 * one loop): h(i) = link(theta . x_i) (a collect, stored to d_h unless NULL) and
 * grad_j = sum_i (h(i) - y_i) * x_ij.  The link is the loop body's own scalar expression of the
 * dot t, compiled to dlx_link_code (registers r[0] = t, r[dst] = op(r[a], r[b]) / imm; IEEE
 * round-to-nearest, no contraction): the reference op set has no exp, so staged programs carry
 * e.g. softsign t / (1 + |t|), and the MathExp extension gives the sigmoid. */
#define DLX_LINK_MAX_CODE 16
#define DLX_LINK_MAX_REGS 8
enum { DLX_LINK_CONST = 0, DLX_LINK_ADD, DLX_LINK_SUB, DLX_LINK_MUL, DLX_LINK_DIV, DLX_LINK_ABS,
       DLX_LINK_EXP, DLX_LINK_SQRT };
typedef struct {
  int32_t n, out;
  uint8_t op[DLX_LINK_MAX_CODE], dst[DLX_LINK_MAX_CODE], a[DLX_LINK_MAX_CODE], b[DLX_LINK_MAX_CODE];
  double imm[DLX_LINK_MAX_CODE];
} dlx_link_code;
/* how dlx_rowdot_link_grad evaluates a link code: 1 = the sigmoid 1 / (1 + exp(0 - t)), 2 = the
 * softsign t / (1 + |t|) (fixed functions, bit-identical to interpreting the code), 0 = the
 * interpreted code */
int dlx_link_kind(const dlx_link_code* h_link);
int dlx_rowdot_link_grad(const double* d_x, const int64_t* d_y, int64_t n, int32_t d,
                         const double* d_theta, const dlx_link_code* h_link, double* d_h,
                         double* d_grad, void* d_workspace, size_t workspace_bytes,
                         dlx_stream_t stream);
/* theta_j -= alpha * grad_j */
int dlx_axpy_inplace(double* d_theta, const double* d_grad, double alpha, int64_t n,
                     dlx_stream_t stream);

/* ---- bucket row sums: the keyed multi-sum multiloop (GDA pass 1's shape: a count and d
 *      column sums per bucket, each a reduce predicated on key(i) == b, loops.cpp:111-174) ---- */
/* For t < nbuckets: d_counts[t] = #{i : keys[i] == h_buckets[t]},
 * d_sums[t*d + j] = sum over those i of x[i*d + j].  x: n*d row-major fp64, keys: n int64.
 * One read of x per 4 (d <= 64), 2 (d <= 128) or 1 (d <= 256) buckets; d > 256 raises
 * DLX_ERR_GENERATION.  Deterministic (fixed-shape per-CTA partials, combine.cu). */
size_t dlx_bucket_rowsum_workspace_bytes(int64_t n, int32_t d, int32_t nbuckets);
int dlx_bucket_rowsum(const double* d_x, const int64_t* d_keys, int64_t n, int32_t d,
                      const int64_t* h_buckets, int32_t nbuckets, int64_t* d_counts, double* d_sums,
                      void* d_workspace, size_t workspace_bytes, dlx_stream_t stream);

/* ---- GDA ----------------------------------------------------------------- */
/* pass 1 (1 + 2d predicated reduces keyed on y): n1 = #{y==1}, sum0/sum1 per class. */
size_t dlx_gda_workspace_bytes(int64_t n, int32_t d);
int dlx_gda_pass1(const double* d_x, const int64_t* d_y, int64_t n, int32_t d, int64_t* d_n1,
                  double* d_sum0, double* d_sum1, void* d_workspace, size_t workspace_bytes,
                  dlx_stream_t stream);
/* mu0 = sum0/(n - n1), mu1 = sum1/n1 (on device; n = the GLOBAL sample count) */
int dlx_gda_means(const int64_t* d_n1, const double* d_sum0, const double* d_sum1,
                  int64_t n_total, int32_t d, double* d_mu0, double* d_mu1, dlx_stream_t stream);
/* pass 2 (d*d reduces): S[a*d+b] = sum_i (x_ia - mu_{y_i,a}) (x_ib - mu_{y_i,b}) */
/* Single-pass GDA fit (d <= 64): n1, mu0, mu1 and S from ONE read of x.  The scatter is
 * accumulated around a shift (the class means of the first <= 64 rows) and corrected by the
 * rank-1 terms sd_c sd_c^T / n_c; when the correction cancels more than 99 % of a diagonal
 * entry, pass 2 on the exact means runs instead (decided on the device, no host sync).
 * Results match dlx_gda_pass1 + dlx_gda_means + dlx_gda_pass2 to rtol 1e-9. */
size_t dlx_gda_fit_workspace_bytes(int64_t n, int32_t d);
int dlx_gda_fit(const double* d_x, const int64_t* d_y, int64_t n, int32_t d, int64_t* d_n1,
                double* d_mu0, double* d_mu1, double* d_scatter, void* d_workspace,
                size_t workspace_bytes, dlx_stream_t stream);
/* Sharded fit: combine the ranks' dlx_gda_fit results.  d_table = world rows of
 * (n0, n1, mu0[d], mu1[d]) as fp64, summed across ranks (rank r fills row r, zeros elsewhere);
 * d_scatter = the sum of the ranks' S on input, the global S on output (pooled-scatter
 * identity, between-rank term from mean differences); writes the global n1, mu0, mu1. */
int dlx_gda_combine_ranks(const double* d_table, int32_t world, int32_t d, double* d_scatter,
                          int64_t* d_n1, double* d_mu0, double* d_mu1, dlx_stream_t stream);
/* 1 if the last dlx_gda_fit on this workspace took the exact-means fallback (synchronous). */
int dlx_gda_fit_last_fallback(const void* d_workspace, int64_t n, int32_t d, int* h_fallback);
/* Which first pass dlx_gda_fit runs for these inputs (host-side, no launch): 2 = the int8
 * tensor-core fit (d = 64, 16-byte aligned x / y, <= 2^17 rows per CTA, DLX_GDA_I8 != 0),
 * 1 = the k-split DMMA fit (d = 64, aligned), 0 = the row-block DMMA kernel. */
int dlx_gda_fit_path(const void* d_x, const void* d_y, int64_t n, int32_t d, int* h_path);
int dlx_gda_pass2(const double* d_x, const int64_t* d_y, int64_t n, int32_t d,
                  const double* d_mu0, const double* d_mu1, double* d_scatter, void* d_workspace,
                  size_t workspace_bytes, dlx_stream_t stream);

/* Vector[Int] from the int32 device assignments (reference Int is int64, types.hpp:11-20). */
int dlx_widen_i32_i64(const int32_t* d_in, int64_t n, int64_t* d_out, dlx_stream_t stream);

/* ---- generic Collect / Reduce families (map, zipWith, sum, count_where, mean/variance) -- */
int dlx_map_axpy(double a, const double* d_x, const double* d_y, int64_t n, double* d_out,
                 dlx_stream_t stream);
size_t dlx_reduce_workspace_bytes(int64_t n);
int dlx_reduce_sum_f64(const double* d_x, int64_t n, double* d_out, void* d_workspace,
                       size_t workspace_bytes, dlx_stream_t stream);
int dlx_reduce_sum_i64(const int64_t* d_x, int64_t n, int64_t* d_out, void* d_workspace,
                       size_t workspace_bytes, dlx_stream_t stream);
/* fused mean_variance loop: out[0] = sum x, out[1] = sum x*x */
int dlx_reduce_sum_sumsq_f64(const double* d_x, int64_t n, double* d_out2, void* d_workspace,
                             size_t workspace_bytes, dlx_stream_t stream);
/* count_where(thr < x[i]) */
int dlx_reduce_count_gt_f64(const double* d_x, int64_t n, double thr, int64_t* d_out,
                            void* d_workspace, size_t workspace_bytes, dlx_stream_t stream);

/* ---- multi-GPU: one process per GPU, sample-sharded, partial activation records summed
 *      with NCCL allReduce over NVLink --------------------------------------- */
#define DLX_COMM_ID_BYTES 128
typedef struct dlx_comm_s* dlx_comm_t;
int dlx_comm_unique_id(uint8_t* h_id /* DLX_COMM_ID_BYTES */);
int dlx_comm_init(dlx_comm_t* comm, const uint8_t* h_id, int nranks, int rank);
int dlx_comm_destroy(dlx_comm_t comm);
/* in-place sum allreduce; dtype: 0 = fp64, 1 = int64 */
int dlx_comm_allreduce_sum(dlx_comm_t comm, void* d_buf, int64_t count, int dtype,
                           dlx_stream_t stream);
/* Several partial records reduced by one fused NCCL launch (ncclGroupStart/End): bufs[i] holds
 * counts[i] elements of dtypes[i] (0 = f64, 1 = i64), each summed in place across ranks. */
int dlx_comm_allreduce_sum_group(dlx_comm_t comm, void* const* d_bufs, const int64_t* counts,
                                 const int* dtypes, int nbufs, dlx_stream_t stream);

/* ---- multi-GPU, peer memory: one-shot allreduce of a partial record fused with its update
 *      (peer.cu).  Each rank allocates an exchange buffer (dlx_peer_alloc, exported as a CUDA
 *      IPC handle), opens every peer's handle (dlx_peer_open) and passes all nranks buffer
 *      pointers (its own at index rank) to dlx_peer_allreduce.  The record is `items` items of
 *      `ni` int64 values (d_counts, items x ni) and `nf` fp64 values (d_sums, items x nf); every
 *      rank folds the per-rank records in ascending rank order (bit-identical on all ranks) and
 *      overwrites its local record with the sum.  epilogue: 0 none; 1 k-means update
 *      d_out[c*nf+j] = sums[c][j] / (double)counts[c] (ni == 1); 2 BGD step
 *      d_out[i] = d_out[i] - alpha * sums[i].  All ranks must issue the same sequence of calls. */
#define DLX_PEER_HANDLE_BYTES 64
int dlx_peer_alloc(int64_t bytes, void** d_ptr, uint8_t* h_handle /* DLX_PEER_HANDLE_BYTES */);
int dlx_peer_open(const uint8_t* h_handle, void** d_ptr);
int dlx_peer_close(void* d_ptr);
int dlx_peer_free(void* d_ptr);
int dlx_peer_allreduce(void* const* h_bufs, int nranks, int rank, int64_t cap_bytes, int64_t items,
                       int ni, int nf, int64_t* d_counts, double* d_sums, int epilogue,
                       double* d_out, double alpha, dlx_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* DLX_H_ */
