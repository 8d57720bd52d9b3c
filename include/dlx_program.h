/*
 * dlx_program.h — C ABI of the multiloop program executor (paper_1109_0778_b200/csrc/program.cpp).
 *
 * The drop-in replacement for the reference's execution entry points, which the reference
 * declares but does not implement:
 *     RunResult interpret(const minic::Program&, uint64_t seed)          (interp.hpp:10)
 *     executeDEG(deg, kernels, workers, chunks) / scheduleDEG(deg, workers)
 * Input: a "dlx-program/1" descriptor — the scheduled, fused stagekit graph serialised by
 * the reference-side adapter (integration/stagekit_dlx.cpp): every live statement, every
 * scheduled block in order, each ParallelLoop's LoopPayload (node.hpp:60-81) with its live
 * elems, and the DEG of build_kernels (codegen.cpp:497-567).  Root-block statements run in
 * schedule order; scalar single-task kernels on the host, synthetic vector sources on the
 * device (reference Rng, shared draw counter in program order), and every ParallelLoop as
 * one of the executor's sm_100a multiloop kernels.  Loops no kernel can lower fail with
 * DLX_ERR_GENERATION (StagingError::GenerationFailed, codegen.cpp:66-71) — no CPU fallback.
 */
#ifndef DLX_PROGRAM_H_
#define DLX_PROGRAM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Runs the program on `device`.  On success *out_text holds the printed output (one line per
 * Print, format_double for doubles: expr.cpp:11-22) and *out_report a JSON report (one
 * entry per root loop: the lowering family chosen and its launches).  Both are allocated
 * here and released with dlx_string_free.  Returns DLX_OK / DLX_ERR_GENERATION /
 * DLX_ERR_TRAP / DLX_ERR_CUDA / DLX_ERR_ARG; dlx_last_error() has the message. */
int dlx_program_run(const char* program_json, uint64_t seed, int device, char** out_text,
                    char** out_report);
void dlx_string_free(char* s);

#ifdef __cplusplus
}
#endif
#endif /* DLX_PROGRAM_H_ */
