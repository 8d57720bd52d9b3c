// jit.hpp — run-time compilation of generated multiloop kernels (the CUDA target's rendering of
// one fused loop body into ONE kernel, north_star: "each fused loop body becomes a single
// templated kernel").  NVRTC (dlopen'ed: libnvrtc.so.12, the CUDA toolkit's) compiles the source
// the lowering generates straight to an sm_100a cubin; the cubin is loaded with the runtime's
// library API (cudaLibraryLoadData: context-independent, so one load serves every device).
// Modules are cached per process by source text, so a program handle executed again, a second
// handle of the same program, or another loop with an identical body never recompiles.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

namespace dlx {

struct JitModule {
  cudaLibrary_t lib = nullptr;
  std::vector<cudaKernel_t> kernels;   // in the order of the names passed to jit_compile
  double compile_ms = 0;               // NVRTC time of the compile that produced it (0: cached)
  size_t cubin_bytes = 0;
};
using JitModuleP = std::shared_ptr<const JitModule>;

// Compiles `src` (or returns the cached module) and resolves `names` (extern "C" kernels).
// Throws Fail(DLX_ERR_GENERATION) with NVRTC's log when the source does not compile, and
// Fail(DLX_ERR_CUDA) when NVRTC cannot be loaded — there is no other path for such a loop.
JitModuleP jit_compile(const std::string& src, const std::vector<std::string>& names);

// compile only (no device needed): throws like jit_compile when the source does not compile
void jit_check(const std::string& src);

// number of NVRTC compiles / cache hits in this process (reported by dlx_jit_stats)
void jit_counts(long long* compiles, long long* hits);

}  // namespace dlx
