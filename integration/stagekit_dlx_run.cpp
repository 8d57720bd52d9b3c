// stagekit_dlx_run.cpp — run_on_b200 (see stagekit_dlx.hpp): links the executor's C ABI.
#include <stdexcept>

#include "stagekit_dlx.hpp"
#include "../include/dlx.h"
#include "../include/dlx_program.h"

// The call a stagekit `run` pipeline makes instead of interpret()/executeDEG().

namespace stagekit_dlx {

stagekit::RunResult run_on_b200(const stagekit::Graph& g, const stagekit::Schedule& s,
                                uint64_t seed, int device) {
  const std::string prog = to_dlx_program(g, s);
  char* text = nullptr;
  char* report = nullptr;
  const int rc = dlx_program_run(prog.c_str(), seed, device, &text, &report);
  if (rc == DLX_ERR_GENERATION)
    throw stagekit::StagingError(stagekit::StagingError::Kind::GenerationFailed, dlx_last_error());
  if (rc == DLX_ERR_TRAP) {
    const std::string m = dlx_last_error();
    throw stagekit::TrapError(m.find("DivByZero") != std::string::npos
                                  ? stagekit::TrapError::Kind::DivByZero
                                  : stagekit::TrapError::Kind::IndexOutOfBounds,
                              m);
  }
  if (rc != DLX_OK) throw std::runtime_error(dlx_last_error());
  stagekit::RunResult r;
  r.output = text;
  dlx_string_free(text);
  dlx_string_free(report);
  return r;
}

}  // namespace stagekit_dlx
