// fuse.hpp — the executor's linear-time multiloop fusion pass (staging at
// production shapes).  A descriptor serialised from an UNFUSED stagekit graph carries
// "fusion": "executor" (integration/stagekit_dlx.cpp::to_dlx_program_unfused); parse_program
// then runs this pass, which fuses ParallelLoops with the reference's rules (horizontal, and
// vertical through VectorLength with contraction: proj/src/fusion.cpp:170-288, 204-210) in one
// walk per statement list instead of the reference's clone-the-graph-per-pair fixpoint.
#pragma once

#include "program_ir.hpp"

namespace dlx {

// Fuses in place; returns the number of fused loop pairs.
int fuse_loops_linear(Program& p);

}  // namespace dlx
