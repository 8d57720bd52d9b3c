// stagekit_dlx.hpp — the reference-side binding: what a stagekit maintainer adds so that the
// `run` path executes on the B200 executor instead of the missing interpreter/executor.
//
// The reference declares (but never implements) the execution entry points
//     RunResult interpret(const minic::Program&, uint64_t seed)        (interp.hpp:10)
//     executeDEG(deg, kernels, workers, chunks) / scheduleDEG(deg, ...)
// This adapter replaces both: it serialises the scheduled, fused graph (the same inputs
// run_codegen consumes: Graph + Schedule, codegen.hpp:53) into the executor's multiloop
// descriptor ("dlx-program/1" JSON: every live statement, every scheduled block in order,
// each ParallelLoop's LoopPayload with its live elems, and the DEG kernels of
// build_kernels), and hands it to dlx_program_run (include/dlx_program.h).
#pragma once

#include <cstdint>
#include <string>

#include "stagekit/codegen.hpp"
#include "stagekit/graph.hpp"
#include "stagekit/runtime.hpp"
#include "stagekit/schedule.hpp"

namespace stagekit_dlx {

// Serialise a scheduled graph (call with a schedule built with motion off).
// with_deg = false leaves the DEG out (the executor does not need it; unfused production-shape
// programs have quadratically many anti-dependence entries); executor_fusion marks a graph the
// reference's fuse_loops has not run on, so the executor fuses its root loops (csrc/fuse.cpp).
std::string to_dlx_program(const stagekit::Graph& g, const stagekit::Schedule& s, bool with_deg = true,
                           bool executor_fusion = false);

// The production-shape path: stage, build_schedule (motion off), and
// serialise WITHOUT the reference's fuse_loops (quadratic: one clone of the whole graph and one
// rebuilt schedule per fused pair, fusion.cpp:170-288) — the executor fuses the root loops in
// one linear pass instead.  No DEG.
std::string to_dlx_program_unfused(const stagekit::Graph& g, const stagekit::Schedule& s);

// Execute on the B200 executor through the C ABI; mirrors interpret()'s result shape.
// Throws stagekit::StagingError(GenerationFailed) for loops the executor cannot lower and
// stagekit::TrapError for runtime traps, like the reference's own paths would.
stagekit::RunResult run_on_b200(const stagekit::Graph& g, const stagekit::Schedule& s,
                                uint64_t seed, int device = 0);

}  // namespace stagekit_dlx
