/*
 * dlx_program.h — C ABI of the multiloop program executor (paper_1109_0778_b200/csrc/program.cpp).
 *
 * The drop-in replacement for the reference's execution entry points, which the reference
 * declares but does not implement:
 *     RunResult interpret(const minic::Program&, uint64_t seed)          (interp.hpp:10)
 *     executeDEG(deg, kernels, workers, chunks) / scheduleDEG(deg, workers)
 *     struct RunResult { std::string output; Value result; }             (runtime.hpp:100-103)
 * Input: a "dlx-program/1" descriptor — the scheduled, fused stagekit graph serialised by
 * the reference-side adapter (integration/stagekit_dlx.cpp): every live statement, every
 * scheduled block in order, each ParallelLoop's LoopPayload (node.hpp:60-81) with its live
 * elems, and the DEG of build_kernels (codegen.cpp:497-567).  Root-block statements run in
 * schedule order; scalar single-task kernels on the host, synthetic vector sources on the
 * device (reference Rng, shared draw counter in program order), and every ParallelLoop as
 * one of the executor's sm_100a multiloop kernels.  Loops no kernel can lower fail with
 * DLX_ERR_GENERATION (StagingError::GenerationFailed, codegen.cpp:66-71) — no CPU fallback.
 *
 * Two ways in:
 *   - dlx_program_create once (parse + static analysis), then dlx_program_execute any number of
 *     times (lowerings are cached per loop statement in the handle), dlx_program_destroy;
 *   - dlx_program_run: one-shot convenience (parsed descriptors cached by content).
 * A handle may be executed by one thread at a time.
 */
#ifndef DLX_PROGRAM_H_
#define DLX_PROGRAM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dlx_program_s* dlx_program_t;

/* element types of program values (reference Ty, types.hpp:11-20) */
enum { DLX_VAL_UNIT = 0, DLX_VAL_INT = 1, DLX_VAL_DOUBLE = 2, DLX_VAL_BOOL = 3, DLX_VAL_STR = 4,
       DLX_VAL_VECTOR = 5 };

/* Caller-supplied data for a VectorRand / VectorRandInt statement (the staged program's
 * synthetic source): the statement `sym` takes these n elements instead of drawing them (the
 * shared draw counter still advances by n, so every other random vector is unchanged).
 * elem: DLX_VAL_DOUBLE for VectorRand, DLX_VAL_INT (int64) for VectorRandInt.  Exactly one of
 * h_data (host memory, copied to the device during the run; pinned memory copies fastest) and
 * d_data (device memory on the execution device, used in place: not copied, not freed) is set. */
typedef struct {
  int32_t sym;
  int32_t elem;
  int64_t n;
  const void* h_data;
  void* d_data;
} dlx_program_input;

enum {
  DLX_EXEC_SERIAL = 1, /* complete every loop before the next statement (no DEG overlap) */
  DLX_EXEC_DRYRUN = 2, /* no device work: lower every loop and report the chosen families */
  DLX_EXEC_NOCACHE = 4 /* re-lower every loop (ignore the handle's lowering cache) */
};

/* ExecOptions: seed of the program's Rng, devices, input bindings, flags.
 * ndevices <= 1 runs on devices[0] (or device 0 when devices is NULL). */
typedef struct {
  uint64_t seed;
  int32_t ndevices;
  const int32_t* devices;
  int32_t ninputs;
  const dlx_program_input* inputs;
  int32_t flags;
} dlx_exec_options;

/* RunResult: the printed text, the per-loop lowering report, and the program's result Value.
 * A vector result is copied to host memory (vec_data: vec_len elements of vec_elem). */
typedef struct {
  char* text;
  char* report;
  int32_t kind;      /* DLX_VAL_* */
  int64_t i;         /* INT, BOOL (0/1) */
  double d;          /* DOUBLE */
  char* s;           /* STR; also the formatted value of every kind */
  int32_t vec_elem;  /* VECTOR: DLX_VAL_INT / DLX_VAL_DOUBLE / DLX_VAL_BOOL (1 byte) */
  int64_t vec_len;
  void* vec_data;
} dlx_run_result;

/* Returns DLX_OK / DLX_ERR_ARG (malformed descriptor); dlx_last_error() has the message. */
int dlx_program_create(const char* program_json, size_t len, dlx_program_t* out);
int dlx_program_destroy(dlx_program_t program);
/* Executes the program.  opts may be NULL (seed 1, device 0).  On DLX_OK *out is filled and
 * must be released with dlx_run_result_free.  Errors: DLX_ERR_GENERATION / DLX_ERR_TRAP /
 * DLX_ERR_CUDA / DLX_ERR_ARG. */
int dlx_program_execute(dlx_program_t program, const dlx_exec_options* opts, dlx_run_result* out);
void dlx_run_result_free(dlx_run_result* r);

/* One-shot: parse (cached by content), execute with seed on device.  On success *out_text holds
 * the printed output (one line per Print, format_double for doubles: expr.cpp:11-22) and
 * *out_report the JSON report (one entry per executed root loop).  Both released with
 * dlx_string_free. */
int dlx_program_run(const char* program_json, uint64_t seed, int device, char** out_text,
                    char** out_report);
void dlx_string_free(char* s);

#ifdef __cplusplus
}
#endif
#endif /* DLX_PROGRAM_H_ */
