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
  dlx_program_t h = nullptr;
  int rc = dlx_program_create(prog.data(), prog.size(), &h);
  dlx_run_result out{};
  if (rc == DLX_OK) {
    dlx_exec_options o{};
    o.seed = seed;
    o.ndevices = 1;
    o.devices = &device;
    rc = dlx_program_execute(h, &o, &out);
    dlx_program_destroy(h);
  }
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
  r.output = out.text;
  // RunResult.result (runtime.hpp:100-103): the program's result Value
  switch (out.kind) {
    case DLX_VAL_INT: r.result = stagekit::Value(static_cast<int64_t>(out.i)); break;
    case DLX_VAL_DOUBLE: r.result = stagekit::Value(out.d); break;
    case DLX_VAL_BOOL: r.result = stagekit::Value(out.i != 0); break;
    case DLX_VAL_STR: r.result = stagekit::Value(std::string(out.s)); break;
    case DLX_VAL_VECTOR: {
      auto v = std::make_shared<stagekit::VecData>();
      const size_t n = static_cast<size_t>(out.vec_len);
      if (out.vec_elem == DLX_VAL_DOUBLE) {
        v->kind = stagekit::VecData::Elem::F64;
        v->dv.assign(static_cast<const double*>(out.vec_data), static_cast<const double*>(out.vec_data) + n);
      } else if (out.vec_elem == DLX_VAL_BOOL) {
        v->kind = stagekit::VecData::Elem::Bool;
        v->bv.assign(static_cast<const uint8_t*>(out.vec_data), static_cast<const uint8_t*>(out.vec_data) + n);
      } else {
        v->kind = stagekit::VecData::Elem::I64;
        v->iv.assign(static_cast<const int64_t*>(out.vec_data), static_cast<const int64_t*>(out.vec_data) + n);
      }
      r.result = stagekit::Value(v);
      break;
    }
    default: break;   // Unit
  }
  dlx_run_result_free(&out);
  return r;
}

}  // namespace stagekit_dlx
