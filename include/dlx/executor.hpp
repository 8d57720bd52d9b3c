// executor.hpp — C++ API of the B200 multiloop program executor (host side of the drop-in).
//
// Mirrors the reference's execution interface and error behaviour:
//   stagekit::RunResult {output, result}                        (runtime.hpp:100-103)
//   RunResult interpret(const minic::Program&, uint64_t seed)   (interp.hpp:10, body absent)
//   StagingError::GenerationFailed ("don't know how to generate code for", codegen.cpp:66-71)
//   TrapError {DivByZero, IndexOutOfBounds}                     (errors.hpp:46-67)
// The program is the "dlx-program/1" descriptor of a scheduled, fused stagekit graph
// (integration/stagekit_dlx.cpp).  The C ABI over this is include/dlx_program.h.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

namespace dlx {

struct RunResult {
  std::string output;  // printed text, one line per Print (format_double for doubles)
  std::string result;  // formatted program result (Unit -> "()")
  std::string report;  // JSON: per root loop, the lowering family and its launch
};

struct GenerationFailed : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct TrapError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Runs the descriptor on `device`.  Throws GenerationFailed / TrapError / std::runtime_error.
RunResult run_program(const std::string& program_json, uint64_t seed, int device = 0);

// Shortest round-trip fp64 text with ".0" for integral values (expr.cpp:11-22).
std::string format_double(double x);

}  // namespace dlx
