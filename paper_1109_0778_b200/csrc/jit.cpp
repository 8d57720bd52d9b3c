// jit.cpp — NVRTC compile + runtime library load of generated multiloop kernels (see jit.hpp).
#include "jit.hpp"

#include <dlfcn.h>

#include <chrono>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "program_ir.hpp"

namespace dlx {

namespace {

// the few NVRTC entry points used (nvrtc.h, CUDA 12): declared here so the library is opened at
// first use rather than linked (a process that never meets a generic loop never loads it)
typedef int nvrtcResult_t;
typedef struct _nvrtcProgram* nvrtcProgram_t;
struct Nvrtc {
  nvrtcResult_t (*CreateProgram)(nvrtcProgram_t*, const char*, const char*, int, const char* const*, const char* const*);
  nvrtcResult_t (*CompileProgram)(nvrtcProgram_t, int, const char* const*);
  nvrtcResult_t (*GetProgramLogSize)(nvrtcProgram_t, size_t*);
  nvrtcResult_t (*GetProgramLog)(nvrtcProgram_t, char*);
  nvrtcResult_t (*GetCUBINSize)(nvrtcProgram_t, size_t*);
  nvrtcResult_t (*GetCUBIN)(nvrtcProgram_t, char*);
  nvrtcResult_t (*DestroyProgram)(nvrtcProgram_t*);
  const char* (*GetErrorString)(nvrtcResult_t);
  bool ok = false;
  std::string why;
};

const Nvrtc& nvrtc() {
  static Nvrtc api = [] {
    Nvrtc a{};
    void* h = nullptr;
    const char* env = std::getenv("DLX_NVRTC_LIB");
    for (const char* name : {env, "libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so"}) {
      if (name && (h = dlopen(name, RTLD_NOW | RTLD_LOCAL))) break;
    }
    if (!h) {
      a.why = "cannot load NVRTC (libnvrtc.so.12; set DLX_NVRTC_LIB)";
      return a;
    }
#define DLX_NVRTC(f) a.f = reinterpret_cast<decltype(a.f)>(dlsym(h, "nvrtc" #f))
    DLX_NVRTC(CreateProgram);
    DLX_NVRTC(CompileProgram);
    DLX_NVRTC(GetProgramLogSize);
    DLX_NVRTC(GetProgramLog);
    DLX_NVRTC(GetCUBINSize);
    DLX_NVRTC(GetCUBIN);
    DLX_NVRTC(DestroyProgram);
    DLX_NVRTC(GetErrorString);
#undef DLX_NVRTC
    a.ok = a.CreateProgram && a.CompileProgram && a.GetProgramLogSize && a.GetProgramLog && a.GetCUBINSize &&
           a.GetCUBIN && a.DestroyProgram && a.GetErrorString;
    if (!a.ok) a.why = "NVRTC library lacks nvrtcGetCUBIN (CUDA >= 11.1 needed)";
    return a;
  }();
  return api;
}

std::mutex g_mu;
std::unordered_map<std::string, JitModuleP> g_cache;   // (names + source) -> module
long long g_compiles = 0, g_hits = 0;

}  // namespace

// NVRTC: source -> sm_100a cubin (throws on failure)
static std::string nvrtc_cubin(const std::string& src, double* ms) {
  const Nvrtc& api = nvrtc();
  if (!api.ok) throw Fail(DLX_ERR_CUDA, "generated multiloop kernel: " + api.why);
  const auto t0 = std::chrono::steady_clock::now();
  nvrtcProgram_t prog = nullptr;
  int rc = api.CreateProgram(&prog, src.c_str(), "dlx_multiloop.cu", 0, nullptr, nullptr);
  if (rc != 0) throw Fail(DLX_ERR_CUDA, std::string("nvrtcCreateProgram: ") + api.GetErrorString(rc));
  // sm_100a cubin; no FMA contraction: every fp64 op rounds on its own, as the reference's MiniC
  // evaluates `acc = acc + d * d` (the generated code also spells the rounding intrinsics out)
  const char* opts[] = {"-arch=sm_100a", "-std=c++17", "--fmad=false", "-lineinfo", "-default-device"};
  rc = api.CompileProgram(prog, static_cast<int>(sizeof(opts) / sizeof(opts[0])), opts);
  size_t log_n = 0;
  api.GetProgramLogSize(prog, &log_n);
  std::string log(log_n, '\0');
  if (log_n) api.GetProgramLog(prog, &log[0]);
  if (rc != 0) {
    api.DestroyProgram(&prog);
    throw Fail(DLX_ERR_GENERATION, "GenerationFailed: generated multiloop kernel does not compile: " + log.substr(0, 2000));
  }
  size_t n = 0;
  api.GetCUBINSize(prog, &n);
  std::string cubin(n, '\0');
  api.GetCUBIN(prog, &cubin[0]);
  api.DestroyProgram(&prog);
  if (ms) *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return cubin;
}

void jit_check(const std::string& src) { nvrtc_cubin(src, nullptr); }

JitModuleP jit_compile(const std::string& src, const std::vector<std::string>& names) {
  std::string key;
  for (const std::string& n : names) key += n + ",";
  key += "\n" + src;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_cache.find(key);
    if (it != g_cache.end()) {
      ++g_hits;
      return it->second;
    }
  }
  auto m = std::make_shared<JitModule>();
  const std::string cubin = nvrtc_cubin(src, &m->compile_ms);
  m->cubin_bytes = cubin.size();
  cudaError_t e = cudaLibraryLoadData(&m->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  if (e != cudaSuccess) throw Fail(DLX_ERR_CUDA, std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e));
  for (const std::string& nm : names) {
    cudaKernel_t k = nullptr;
    e = cudaLibraryGetKernel(&k, m->lib, nm.c_str());
    if (e != cudaSuccess) throw Fail(DLX_ERR_CUDA, "cudaLibraryGetKernel(" + nm + "): " + cudaGetErrorString(e));
    m->kernels.push_back(k);
  }
  std::lock_guard<std::mutex> lk(g_mu);
  ++g_compiles;
  auto [it, fresh] = g_cache.emplace(key, m);   // a racing thread's module wins; ours is dropped
  return it->second;
}

void jit_counts(long long* compiles, long long* hits) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (compiles) *compiles = g_compiles;
  if (hits) *hits = g_hits;
}

}  // namespace dlx
