// program.cpp — the multiloop program executor: the B200 replacement for the reference's
// missing interpret() / executeDEG() (interp.hpp:10).  See
// include/dlx_program.h for the contract and include/dlx/executor.hpp for the C++ API.
//
// Execution model (mirrors SPEC.md's runtime module):
//   * root-block statements run in schedule order (the DEG's data and anti-dependence edges
//     are respected by construction: build_kernels derives them from this same order);
//   * single-task scalar statements (Op set node.hpp:15-27, IfThenElse, While, Var*) are
//     evaluated on the host with the reference semantics: Int wraps (graph.cpp:10-21), Int
//     division by zero traps, Double is IEEE;
//   * vectors are device-resident (DenseVector mirrors of VecData, runtime.hpp:44-72);
//     VectorRand / VectorRandInt draw from one Rng(seed) in program order on the device;
//   * every ParallelLoop (LoopPayload, node.hpp:76-81) is lowered by the CUDA target: its
//     live elems are symbolically evaluated into an expression DAG (loads at affine indices,
//     scalar ops, nested reduces), then matched against the specialised families (fused
//     k-means, bucket counts, GDA passes 1/2) and otherwise compiled to the generic multiloop
//     kernel's bytecode (vm.cu).  Anything else raises GenerationFailed.
#include <cuda_runtime.h>

#include <algorithm>
#include <tuple>

#include <charconv>
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <json.hpp>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <variant>
#include <vector>

#include "../../include/dlx.h"
#include "../../include/dlx/executor.hpp"
#include "../../include/dlx_program.h"
#include "../../include/dlx_vm.h"

namespace dlx {

void set_error(const char* fmt, ...);

std::string format_double(double x) {
  if (std::isnan(x)) return "nan";
  if (std::isinf(x)) return x > 0 ? "inf" : "-inf";
  char buf[64];
  auto res = std::to_chars(buf, buf + sizeof(buf), x);
  std::string s(buf, res.ptr);
  if (s.find('.') == std::string::npos && s.find('e') == std::string::npos) s += ".0";
  return s;
}

namespace {

using json = nlohmann::json;

// ---- errors --------------------------------------------------------------------------------
struct Fail : std::runtime_error {
  int code;
  Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void gen_fail(const std::string& m) {
  throw Fail(DLX_ERR_GENERATION, "GenerationFailed: " + m);
}
[[noreturn]] void trap(const std::string& m) { throw Fail(DLX_ERR_TRAP, m); }
void ck(int rc) {
  if (rc != DLX_OK) throw Fail(rc, dlx_last_error());
}
void ckc(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Fail(DLX_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- IR (parsed dlx-program/1) ----------------------------------------------------------------
enum class Ty { Int, Double, Bool, Str, Unit, Vector, Var, Other };
struct Type {
  Ty t = Ty::Unit;
  Ty elem = Ty::Unit;  // Vector / Var payload
};
Type parse_type(const std::string& s) {
  auto base = [](const std::string& b) {
    if (b == "Int") return Ty::Int;
    if (b == "Double") return Ty::Double;
    if (b == "Bool") return Ty::Bool;
    if (b == "Str") return Ty::Str;
    if (b == "Unit") return Ty::Unit;
    return Ty::Other;
  };
  Type t;
  if (s.rfind("Vector[", 0) == 0) {
    t.t = Ty::Vector;
    t.elem = base(s.substr(7, s.size() - 8));
  } else if (s.rfind("Var[", 0) == 0) {
    t.t = Ty::Var;
    t.elem = base(s.substr(4, s.size() - 5));
  } else {
    t.t = base(s);
  }
  return t;
}

struct Atom {  // stagekit::Expr: a literal or a symbol
  enum K { Sym, Int, Double, Bool, Str, Unit } k = Unit;
  int sym = -1;
  int64_t i = 0;
  double d = 0;
  bool b = false;
  std::string s;
  Type ty;
};
Atom parse_atom(const json& j) {
  Atom a;
  if (j.contains("t")) a.ty = parse_type(j["t"].get<std::string>());
  if (j.contains("s")) a.k = Atom::Sym, a.sym = j["s"].get<int>();
  else if (j.contains("i")) a.k = Atom::Int, a.i = j["i"].get<int64_t>();
  else if (j.contains("d")) a.k = Atom::Double, a.d = j["d"].get<double>();
  else if (j.contains("b")) a.k = Atom::Bool, a.b = j["b"].get<bool>();
  else if (j.contains("str")) a.k = Atom::Str, a.s = j["str"].get<std::string>();
  return a;
}

struct Elem {
  std::string kind;
  bool live = true;
  int out = -1;
  Type out_ty;
  int elem = -1, cond = -1, combine = -1;
  bool append = false;
  Atom zero;
  int rv_left = -1, rv_right = -1;
};
struct Loop {
  Atom range;
  int index = -1, body = -1;
  std::vector<Elem> elems;
};
struct Stmt {
  int sym = -1;
  std::string op;
  Type ty;
  std::vector<Atom> args;
  std::vector<int> blocks;
  Type aux_ty;
  std::vector<Atom> lits;
  std::shared_ptr<Loop> loop;
};
struct Block {
  std::vector<int> stmts;
  Atom result;
};
struct Program {
  int root = -1;
  std::unordered_map<int, Stmt> stmts;
  std::unordered_map<int, Block> blocks;
};

Program parse_program(const std::string& text) {
  json j = json::parse(text);
  if (j.value("format", "") != "dlx-program/1") throw Fail(DLX_ERR_ARG, "not a dlx-program/1 descriptor");
  Program p;
  p.root = j["root"].get<int>();
  for (auto& [k, v] : j["blocks"].items()) {
    Block b;
    for (auto& s : v["stmts"]) b.stmts.push_back(s.get<int>());
    b.result = parse_atom(v["result"]);
    p.blocks[std::stoi(k)] = std::move(b);
  }
  for (auto& [k, v] : j["stmts"].items()) {
    Stmt s;
    s.sym = std::stoi(k);
    s.op = v["op"].get<std::string>();
    s.ty = parse_type(v["ty"].get<std::string>());
    for (auto& a : v["args"]) s.args.push_back(parse_atom(a));
    if (v.contains("blocks"))
      for (auto& b : v["blocks"]) s.blocks.push_back(b.get<int>());
    if (v.contains("aux_ty")) s.aux_ty = parse_type(v["aux_ty"].get<std::string>());
    if (v.contains("lits"))
      for (auto& l : v["lits"]) s.lits.push_back(parse_atom(l));
    if (v.contains("loop")) {
      auto L = std::make_shared<Loop>();
      const json& jl = v["loop"];
      L->range = parse_atom(jl["range"]);
      L->index = jl["index"].get<int>();
      L->body = jl["body"].get<int>();
      for (auto& je : jl["elems"]) {
        Elem e;
        e.kind = je["kind"].get<std::string>();
        e.live = je["live"].get<bool>();
        e.out = je["out"].get<int>();
        e.out_ty = parse_type(je["out_ty"].get<std::string>());
        e.elem = je["elem"].get<int>();
        e.cond = je["cond"].get<int>();
        e.combine = je["combine"].get<int>();
        e.append = je["append"].get<bool>();
        if (je.contains("zero")) e.zero = parse_atom(je["zero"]);
        e.rv_left = je.value("rv_left", -1);
        e.rv_right = je.value("rv_right", -1);
        L->elems.push_back(std::move(e));
      }
      s.loop = L;
    }
    p.stmts[s.sym] = std::move(s);
  }
  return p;
}

// ---- runtime values ---------------------------------------------------------------------------
// Dry run (DLX_PROGRAM_DRYRUN=1, CPU-only diagnostics): no device memory and no launches; loops
// are still parsed, symbolically evaluated and matched, so the report shows which lowering
// each loop would get.  Printed values are meaningless in a dry run.
static bool g_dry = false;
static bool g_debug = false;  // DLX_PROGRAM_DEBUG=1: why a specialised family did not match
#define MISS(why)                                                        \
  do {                                                                   \
    if (g_debug) fprintf(stderr, "[dlx program] %s: %s\n", __func__, why); \
    return false;                                                        \
  } while (0)
// Device vector.  Small vectors (<= kMirrorBytes: centroids, counts, sums, parameters) keep a
// host mirror so the host statements that read or update them element by element
// (VectorApply / VectorUpdate — e.g. the k*d `mu(c*d+j) = sum / count` updates of a staged
// k-means iteration) cost one transfer per vector instead of one synchronous copy per element:
// the mirror is loaded on the first host read, host writes mark a dirty range, and every device
// launch first flushes dirty ranges (one copy each) and afterwards invalidates the mirrors.
constexpr size_t kMirrorBytes = 64 << 10;
constexpr int64_t kPageElems = 8192;   // read-through page of a large vector (64 KiB of fp64)
bool g_no_mirror = false;   // DLX_PROGRAM_NO_MIRROR=1: per-element transfers (A/B timing only)
bool g_serial = false;      // DLX_PROGRAM_SERIAL=1: complete every loop before the next statement
// The run's main stream (host statements, RNG fills, mirror flushes, frees) and the fence that
// orders the main stream after every in-flight loop before device memory is freed or rewritten.
thread_local cudaStream_t g_main_st = nullptr;
thread_local std::function<void()>* g_fence = nullptr;
struct DevVec {
  void* p = nullptr;
  int64_t n = 0;
  Ty elem = Ty::Double;
  cudaStream_t fst = nullptr;   // stream the buffer is freed on (stream-ordered allocator)
  std::vector<unsigned char> host;
  bool host_valid = false;
  // large vectors: a read-through page of host copies around the last element read (host
  // statements that read x(0), x(1), ... — the k-means centroid initialisation — cost one
  // transfer per page instead of one synchronous copy per element)
  std::vector<unsigned char> page;
  int64_t page_lo = 0;
  bool page_valid = false;
  int64_t dirty_lo = INT64_MAX, dirty_hi = -1;   // [lo, hi) newer on the host than on the device
  ~DevVec() {
    if (!p) return;
    if (g_fence) (*g_fence)();   // a loop still in flight may read this buffer
    cudaFreeAsync(p, fst);
  }
  size_t esize() const { return elem == Ty::Bool ? 1 : 8; }
  bool mirrored() const { return !g_no_mirror && static_cast<size_t>(n) * esize() <= kMirrorBytes; }
};
using VecP = std::shared_ptr<DevVec>;
// vectors created during one run (for flush / invalidate around device launches)
thread_local std::vector<std::weak_ptr<DevVec>>* g_vecs = nullptr;
struct Cell;
using CellP = std::shared_ptr<Cell>;
struct Val {
  std::variant<std::monostate, int64_t, double, bool, std::string, VecP, CellP> v;
  bool is_int() const { return std::holds_alternative<int64_t>(v); }
  bool is_dbl() const { return std::holds_alternative<double>(v); }
  bool is_bool() const { return std::holds_alternative<bool>(v); }
  bool is_vec() const { return std::holds_alternative<VecP>(v); }
  int64_t i() const { return std::get<int64_t>(v); }
  double d() const { return std::get<double>(v); }
  bool b() const { return std::get<bool>(v); }
  const VecP& vec() const { return std::get<VecP>(v); }
};
struct Cell {
  Val v;
};

VecP new_vec(int64_t n, Ty elem, cudaStream_t st, bool zero) {
  auto v = std::make_shared<DevVec>();
  v->n = n;
  v->elem = elem;
  if (g_vecs) g_vecs->push_back(v);
  if (g_dry) return v;
  v->fst = g_main_st;
  ckc(cudaMallocAsync(&v->p, std::max<size_t>(16, static_cast<size_t>(n) * v->esize()), st), "cudaMallocAsync");
  if (zero) ckc(cudaMemsetAsync(v->p, 0, static_cast<size_t>(n) * v->esize(), st), "cudaMemset");
  return v;
}

std::string format_val(const Val& x) {
  if (x.is_int()) return std::to_string(x.i());
  if (x.is_dbl()) return format_double(x.d());
  if (x.is_bool()) return x.b() ? "true" : "false";
  if (auto s = std::get_if<std::string>(&x.v)) return *s;
  if (x.is_vec()) return "<vector of " + std::to_string(x.vec()->n) + ">";
  return "()";
}

// ---- symbolic expressions of loop bodies ------------------------------------------------------
struct SE;
using SEP = std::shared_ptr<SE>;
struct SE {
  enum K { Const, Idx, Inner, Host, Vec, Load, Bin, Un, Sel, Red, RvL, RvR } k;
  Ty ty = Ty::Int;
  std::string op;
  int64_t ci = 0;
  double cd = 0;
  Val host;
  VecP vec;
  int sym = -1;            // Inner: index symbol
  std::vector<SEP> a;      // children (Red: elem, cond, combine)
  int64_t range = 0;       // Red
  Atom zero;               // Red
};
SEP mk(SE::K k, Ty ty) {
  auto s = std::make_shared<SE>();
  s->k = k;
  s->ty = ty;
  return s;
}
bool is_const_int(const SEP& s, int64_t* v = nullptr) {
  if (s->k == SE::Const && s->ty == Ty::Int) {
    if (v) *v = s->ci;
    return true;
  }
  if (s->k == SE::Host && s->host.is_int()) {
    if (v) *v = s->host.i();
    return true;
  }
  return false;
}
bool is_const_dbl(const SEP& s, double* v = nullptr) {
  if (s->k == SE::Const && s->ty == Ty::Double) {
    if (v) *v = s->cd;
    return true;
  }
  if (s->k == SE::Host && s->host.is_dbl()) {
    if (v) *v = s->host.d();
    return true;
  }
  return false;
}

// the same value: one node, or two literal nodes with equal payloads (literals are not shared)
bool same_se(const SEP& x, const SEP& y) {
  if (x == y) return true;
  if (x->k == SE::Const && y->k == SE::Const && x->ty == y->ty)
    return x->ty == Ty::Double ? std::memcmp(&x->cd, &y->cd, 8) == 0 : x->ci == y->ci;
  return false;
}

// affine form a*Idx + b*Inner(sym) + c
struct Affine {
  int64_t a = 0, b = 0, c = 0;
  int inner = -1;
};
std::optional<Affine> affine(const SEP& s) {
  int64_t v;
  if (is_const_int(s, &v)) return Affine{0, 0, v, -1};
  if (s->k == SE::Idx) return Affine{1, 0, 0, -1};
  if (s->k == SE::Inner) return Affine{0, 1, 0, s->sym};
  if (s->k == SE::Bin && (s->op == "Plus" || s->op == "Minus" || s->op == "Times")) {
    auto x = affine(s->a[0]), y = affine(s->a[1]);
    if (!x || !y) return std::nullopt;
    if (x->inner >= 0 && y->inner >= 0 && x->inner != y->inner) return std::nullopt;
    const int inner = x->inner >= 0 ? x->inner : y->inner;
    if (s->op == "Plus") return Affine{x->a + y->a, x->b + y->b, x->c + y->c, inner};
    if (s->op == "Minus") return Affine{x->a - y->a, x->b - y->b, x->c - y->c, inner};
    if (x->a == 0 && x->b == 0) return Affine{x->c * y->a, x->c * y->b, x->c * y->c, inner};
    if (y->a == 0 && y->b == 0) return Affine{y->c * x->a, y->c * x->b, y->c * x->c, inner};
  }
  return std::nullopt;
}

// ---- per-thread, per-device execution resources (kept across runs) ------------------------------
// Loop streams: independent root loops (no data edge between them in the DEG, i.e. neither
// reads a value the other binds) are launched on different streams and their completions are
// deferred, so the kernels overlap each other and the host statements that follow
// (scheduleDEG's concurrent independent kernels).  Results come back through a
// pinned staging arena so the device->host copies stay asynchronous.
constexpr int kLoopStreams = 4;
struct PinnedArena {
  std::vector<std::pair<unsigned char*, size_t>> blocks;   // the last block is the current one
  size_t used = 0;
  void* get(size_t bytes) {
    bytes = (std::max<size_t>(bytes, 1) + 63) & ~size_t{63};
    if (blocks.empty() || used + bytes > blocks.back().second) {
      const size_t sz = std::max<size_t>(bytes, 1 << 20);
      void* h = nullptr;
      ckc(cudaMallocHost(&h, sz), "cudaMallocHost");
      blocks.emplace_back(static_cast<unsigned char*>(h), sz);
      used = 0;
    }
    void* r = blocks.back().first + used;
    used += bytes;
    return r;
  }
  template <class T>
  T* get_n(size_t n) { return static_cast<T*>(get(n * sizeof(T))); }
  void reset() {   // nothing in flight: keep one block, as large as the run needed
    if (blocks.size() > 1) {
      size_t total = 0;
      for (auto& b : blocks) {
        total += b.second;
        cudaFreeHost(b.first);
      }
      blocks.clear();
      void* h = nullptr;
      if (cudaMallocHost(&h, total) == cudaSuccess) blocks.emplace_back(static_cast<unsigned char*>(h), total);
    }
    used = 0;
  }
};
struct DeviceRes {
  cudaStream_t loop[kLoopStreams] = {};
  std::vector<cudaEvent_t> events;   // free list
  PinnedArena pin;
  bool init = false;
};
DeviceRes& device_res(int device) {
  thread_local std::map<int, DeviceRes> res;   // never torn down (process-lifetime streams)
  DeviceRes& r = res[device];
  if (!r.init) {
    for (auto& s : r.loop) ckc(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    cudaMemPool_t pool;   // keep freed blocks of the stream-ordered allocator for the next loops
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      // DLX_POOL_KEEP_GB: bytes the pool keeps mapped across syncs (default 32 GB: remapping an
      // 8 GiB input on every run cost 0.1-1 s per C4 program run, r131)
      const char* kg = getenv("DLX_POOL_KEEP_GB");
      uint64_t keep = kg ? static_cast<uint64_t>(atof(kg) * (1ull << 30)) : (32ull << 30);
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    r.init = true;
  }
  return r;
}

// ---- the executor -------------------------------------------------------------------------------
class Executor {
 public:
  Executor(const Program& p, uint64_t seed, cudaStream_t st, DeviceRes* res)
      : P(p), seed_(seed), st_(st), res_(res), lst_(st) {
    fence_ = [this] { fence(); };
  }

  std::string output;
  json report = json::array();

  Val run() {
    Val v = exec_block(P.root);
    join_all();
    return v;
  }
  std::function<void()> fence_;   // g_fence points here during the run

 private:
  const Program& P;
  uint64_t seed_;
  uint64_t draws_ = 0;
  cudaStream_t st_;
  DeviceRes* res_;
  cudaStream_t lst_;   // stream of the loop being launched
  int64_t launches_ = 0;
  std::unordered_map<int, Val> env_;

  // ---- deferred loop completion (DEG overlap) -----------------------------------------------
  struct Pending {
    cudaEvent_t ev;                 // recorded on the loop's stream after its result copies
    std::function<void()> finish;   // binds the loop's outputs (and raises its traps)
  };
  std::vector<Pending> pending_;   // launch (= program) order
  cudaEvent_t get_event() {
    if (res_->events.empty()) {
      cudaEvent_t e;
      ckc(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
      return e;
    }
    cudaEvent_t e = res_->events.back();
    res_->events.pop_back();
    return e;
  }
  // The loop just enqueued on lst_ binds `outs` when it completes.  Until then the symbols are
  // unbound, so the first statement that reads one of them joins (a data edge of the DEG).
  void defer(const std::vector<int>& outs, std::function<void()> fn) {
    for (int o : outs) env_.erase(o);
    cudaEvent_t ev = get_event();
    ckc(cudaEventRecord(ev, lst_), "cudaEventRecord");
    pending_.push_back(Pending{ev, std::move(fn)});
    if (g_serial) join_all();
  }
  // Device-side ordering only: later main-stream work (frees, host->device rewrites of vectors
  // a pending loop may read: the DEG's anti-dependences) waits for every loop in flight.
  void fence() {
    for (const Pending& p : pending_) cudaStreamWaitEvent(st_, p.ev, 0);
  }
  void join_all() {
    if (pending_.empty()) return;
    std::vector<Pending> pend;
    pend.swap(pending_);
    cudaError_t err = cudaSuccess;
    for (const Pending& p : pend) {
      cudaError_t e = cudaEventSynchronize(p.ev);
      if (err == cudaSuccess) err = e;
      res_->events.push_back(p.ev);
    }
    struct ArenaReset {   // the staged results are consumed (or abandoned on a trap)
      PinnedArena& a;
      ~ArenaReset() { a.reset(); }
    } arena_reset{res_->pin};
    ckc(err, "loop completion");
    for (Pending& p : pend) p.finish();   // program order: the first loop's trap wins
  }
  void* dalloc(size_t bytes) {
    void* p = nullptr;
    ckc(cudaMallocAsync(&p, std::max<size_t>(bytes, 16), lst_), "cudaMallocAsync");
    return p;
  }
  void dfree(void* p) {
    if (p) cudaFreeAsync(p, lst_);
  }
 public:
  std::vector<std::weak_ptr<DevVec>> vecs_;   // every vector of this run (g_vecs points here)
 private:

  // symbolic state of the loop being lowered
  int loop_index_ = -1;
  int64_t dry_n_ = 0;
  std::unordered_map<int, SEP> sym_;

  // ---- host interpretation ----------------------------------------------------------------------
  Val atom(const Atom& a) {
    switch (a.k) {
      case Atom::Sym: {
        auto it = env_.find(a.sym);
        if (it == env_.end() && !pending_.empty()) {
          join_all();
          it = env_.find(a.sym);
        }
        if (it == env_.end()) gen_fail("x" + std::to_string(a.sym) + " referenced before definition");
        return it->second;
      }
      case Atom::Int: return Val{a.i};
      case Atom::Double: return Val{a.d};
      case Atom::Bool: return Val{a.b};
      case Atom::Str: return Val{a.s};
      default: return Val{};
    }
  }

  Val exec_block(int b) {
    const Block& bl = P.blocks.at(b);
    for (int s : bl.stmts) {
      const Stmt& st = P.stmts.at(s);
      try {
        if (st.op == "ParallelLoop") {
          run_loop(st);  // binds every live elem's `out` (elems[0].out is the statement's own sym)
        } else {
          env_[s] = exec_stmt(st);
        }
      } catch (...) {
        join_all();   // a trap of an earlier loop still in flight takes precedence
        throw;
      }
    }
    return atom(bl.result);
  }

  static int64_t wrap(uint64_t v) { return static_cast<int64_t>(v); }

  Val scalar(const std::string& op, const Val& x, const Val& y) {
    if (op == "And") return Val{x.b() && y.b()};
    if (op == "Or") return Val{x.b() || y.b()};
    if (x.is_int() && y.is_int()) {
      const int64_t a = x.i(), b = y.i();
      if (op == "Plus") return Val{wrap(static_cast<uint64_t>(a) + static_cast<uint64_t>(b))};
      if (op == "Minus") return Val{wrap(static_cast<uint64_t>(a) - static_cast<uint64_t>(b))};
      if (op == "Times") return Val{wrap(static_cast<uint64_t>(a) * static_cast<uint64_t>(b))};
      if (op == "Divide") {
        if (b == 0) trap("TrapDivByZero: integer division by zero");
        return Val{(a == INT64_MIN && b == -1) ? a : a / b};
      }
      if (op == "Lt") return Val{a < b};
      if (op == "Eq") return Val{a == b};
    }
    if (x.is_dbl() && y.is_dbl()) {
      const double a = x.d(), b = y.d();
      if (op == "Plus") return Val{a + b};
      if (op == "Minus") return Val{a - b};
      if (op == "Times") return Val{a * b};
      if (op == "Divide") return Val{a / b};
      if (op == "Lt") return Val{a < b};
      if (op == "Eq") return Val{a == b};
    }
    if (op == "Eq") return Val{x.v == y.v};
    gen_fail("don't know how to evaluate " + op);
  }

  // ---- host mirrors of small vectors ------------------------------------------------------
  void load_mirror(const VecP& v) {
    if (v->host_valid) return;
    v->host.resize(static_cast<size_t>(v->n) * v->esize());
    if (!v->host.empty())
      ckc(cudaMemcpyAsync(v->host.data(), v->p, v->host.size(), cudaMemcpyDeviceToHost, st_), "d2h");
    ckc(cudaStreamSynchronize(st_), "sync");
    v->host_valid = true;
  }
  void flush_mirrors() {   // before a device launch: host updates -> device, one copy per vector
    bool any = false;
    for (auto& w : vecs_)
      if (auto v = w.lock())
        if (v->dirty_hi > v->dirty_lo) {
          if (!any) fence();   // WAR: a loop in flight may still read the old contents
          const size_t es = v->esize();
          ckc(cudaMemcpyAsync(static_cast<unsigned char*>(v->p) + v->dirty_lo * es, v->host.data() + v->dirty_lo * es,
                              static_cast<size_t>(v->dirty_hi - v->dirty_lo) * es, cudaMemcpyHostToDevice, st_),
              "h2d");
          v->dirty_lo = INT64_MAX;
          v->dirty_hi = -1;
          any = true;
        }
    if (any) ckc(cudaStreamSynchronize(st_), "sync");   // the mirrors may change right after
  }
  void invalidate_mirrors() {   // after a device launch: any vector may have been written
    size_t live = 0;
    for (auto& w : vecs_)
      if (auto v = w.lock()) {
        v->host_valid = false;
        v->page_valid = false;
        vecs_[live++] = w;
      }
    vecs_.resize(live);
  }

  Val vec_get(const VecP& v, int64_t i) {
    if (i < 0 || i >= v->n) trap("TrapIndexOutOfBounds: index " + std::to_string(i));
    if (g_dry) return v->elem == Ty::Double ? Val{0.5} : v->elem == Ty::Bool ? Val{false} : Val{int64_t{1}};
    if (v->mirrored()) {
      load_mirror(v);
      const unsigned char* h = v->host.data() + static_cast<size_t>(i) * v->esize();
      if (v->elem == Ty::Double) {
        double x;
        std::memcpy(&x, h, 8);
        return Val{x};
      }
      if (v->elem == Ty::Bool) return Val{*h != 0};
      int64_t x;
      std::memcpy(&x, h, 8);
      return Val{x};
    }
    const size_t es = v->esize();
    if (g_no_mirror) {   // A/B: one synchronous copy per element
      v->page_valid = false;
      v->page.resize(es);
      ckc(cudaStreamSynchronize(st_), "sync");
      ckc(cudaMemcpy(v->page.data(), static_cast<unsigned char*>(v->p) + i * es, es, cudaMemcpyDeviceToHost), "d2h");
      v->page_lo = i;
    } else if (!v->page_valid || i < v->page_lo || i >= v->page_lo + static_cast<int64_t>(v->page.size() / es)) {
      const int64_t lo = i & ~(kPageElems - 1), hi = std::min(v->n, lo + kPageElems);
      v->page.resize(static_cast<size_t>(hi - lo) * es);
      ckc(cudaMemcpyAsync(v->page.data(), static_cast<unsigned char*>(v->p) + lo * es, v->page.size(),
                          cudaMemcpyDeviceToHost, st_), "d2h");
      ckc(cudaStreamSynchronize(st_), "sync");
      v->page_lo = lo;
      v->page_valid = true;
    }
    const unsigned char* h = v->page.data() + static_cast<size_t>(i - v->page_lo) * es;
    if (v->elem == Ty::Double) {
      double x;
      std::memcpy(&x, h, 8);
      return Val{x};
    }
    if (v->elem == Ty::Bool) return Val{*h != 0};
    int64_t x;
    std::memcpy(&x, h, 8);
    return Val{x};
  }

  void vec_set(const VecP& v, int64_t i, const Val& x) {
    if (i < 0 || i >= v->n) trap("TrapIndexOutOfBounds: store index " + std::to_string(i));
    if (g_dry) return;
    if (v->mirrored()) {
      load_mirror(v);
      unsigned char* h = v->host.data() + static_cast<size_t>(i) * v->esize();
      if (v->elem == Ty::Double) {
        const double d = x.d();
        std::memcpy(h, &d, 8);
      } else if (v->elem == Ty::Bool) {
        *h = x.b() ? 1 : 0;
      } else {
        const int64_t q = x.i();
        std::memcpy(h, &q, 8);
      }
      v->dirty_lo = std::min(v->dirty_lo, i);
      v->dirty_hi = std::max(v->dirty_hi, i + 1);
      return;
    }
    fence();
    v->page_valid = false;   // the page may hold the old value
    if (v->elem == Ty::Double) {
      const double d = x.d();
      ckc(cudaMemcpyAsync(static_cast<double*>(v->p) + i, &d, 8, cudaMemcpyHostToDevice, st_), "h2d");
    } else if (v->elem == Ty::Bool) {
      const unsigned char b = x.b();
      ckc(cudaMemcpyAsync(static_cast<unsigned char*>(v->p) + i, &b, 1, cudaMemcpyHostToDevice, st_), "h2d");
    } else {
      const int64_t q = x.i();
      ckc(cudaMemcpyAsync(static_cast<int64_t*>(v->p) + i, &q, 8, cudaMemcpyHostToDevice, st_), "h2d");
    }
    ckc(cudaStreamSynchronize(st_), "sync");  // the host value is a stack temporary
  }

  Val exec_stmt(const Stmt& s) {
    const std::string& op = s.op;
    if (op == "Plus" || op == "Minus" || op == "Times" || op == "Divide" || op == "Lt" ||
        op == "Eq" || op == "And" || op == "Or")
      return scalar(op, atom(s.args[0]), atom(s.args[1]));
    if (op == "Not") return Val{!atom(s.args[0]).b()};
    if (op == "MathAbs") {
      Val x = atom(s.args[0]);
      if (x.is_int()) return Val{x.i() < 0 ? wrap(0ull - static_cast<uint64_t>(x.i())) : x.i()};
      return Val{std::fabs(x.d())};
    }
    if (op == "MathSqrt") return Val{std::sqrt(atom(s.args[0]).d())};
    if (op == "ToDouble") return Val{static_cast<double>(atom(s.args[0]).i())};
    if (op == "IfThenElse") return exec_block(atom(s.args[0]).b() ? s.blocks[0] : s.blocks[1]);
    if (op == "While") {
      while (exec_block(s.blocks[0]).b()) exec_block(s.blocks[1]);
      return Val{};
    }
    if (op == "VarAlloc") {
      auto c = std::make_shared<Cell>();
      c->v = atom(s.args[0]);
      return Val{c};
    }
    if (op == "VarRead") return std::get<CellP>(atom(s.args[0]).v)->v;
    if (op == "VarWrite") {
      std::get<CellP>(atom(s.args[0]).v)->v = atom(s.args[1]);
      return Val{};
    }
    if (op == "Print") {
      output += format_val(atom(s.args[0])) + "\n";
      return Val{};
    }
    if (op == "VectorRand" || op == "VectorRandInt") {
      const int64_t n = atom(s.args[0]).i();
      const bool ints = op == "VectorRandInt";
      VecP v = new_vec(n, ints ? Ty::Int : Ty::Double, st_, false);
      if (g_dry) {
      } else if (ints)
        ck(dlx_rng_ints(static_cast<int64_t*>(v->p), n, atom(s.args[1]).i(), seed_, draws_, st_));
      else
        ck(dlx_rng_units(static_cast<double*>(v->p), n, seed_, draws_, st_));
      draws_ += static_cast<uint64_t>(n);
      return Val{v};
    }
    if (op == "VectorNew") {
      const Ty e = s.aux_ty.t;
      if (e != Ty::Int && e != Ty::Double && e != Ty::Bool) gen_fail("vector of " + std::to_string(int(e)));
      return Val{new_vec(atom(s.args[0]).i(), e, st_, true)};
    }
    if (op == "VectorLiteral") {
      const Ty e = s.aux_ty.t == Ty::Double ? Ty::Double : Ty::Int;
      VecP v = new_vec(static_cast<int64_t>(s.lits.size()), e, st_, false);
      std::vector<int64_t> raw(s.lits.size());
      for (size_t q = 0; q < s.lits.size(); ++q) {
        if (e == Ty::Double) {
          const double d = s.lits[q].k == Atom::Double ? s.lits[q].d : static_cast<double>(s.lits[q].i);
          std::memcpy(&raw[q], &d, 8);
        } else {
          raw[q] = s.lits[q].i;
        }
      }
      if (!g_dry) {
        ckc(cudaMemcpyAsync(v->p, raw.data(), raw.size() * 8, cudaMemcpyHostToDevice, st_), "h2d");
        ckc(cudaStreamSynchronize(st_), "sync");
      }
      return Val{v};
    }
    if (op == "VectorLength") return Val{atom(s.args[0]).vec()->n};
    if (op == "VectorApply") return vec_get(atom(s.args[0]).vec(), atom(s.args[1]).i());
    if (op == "VectorUpdate") {
      vec_set(atom(s.args[0]).vec(), atom(s.args[1]).i(), atom(s.args[2]));
      return Val{};
    }
    if (op == "ParallelLoop") return run_loop(s);
    gen_fail("don't know how to generate code for: " + op + " (x" + std::to_string(s.sym) + ")");
  }

  // ---- symbolic evaluation of a loop body ------------------------------------------------------
  SEP sym_atom(const Atom& a) {
    switch (a.k) {
      case Atom::Sym: {
        if (a.sym == loop_index_) return mk(SE::Idx, Ty::Int);
        auto it = sym_.find(a.sym);
        if (it != sym_.end()) return it->second;
        auto e = env_.find(a.sym);
        if (e == env_.end() && !pending_.empty()) {
          join_all();
          e = env_.find(a.sym);
        }
        if (e == env_.end()) gen_fail("loop body reads x" + std::to_string(a.sym) + " before definition");
        const Val& v = e->second;
        if (v.is_vec()) {
          auto s = mk(SE::Vec, v.vec()->elem);
          s->vec = v.vec();
          return s;
        }
        auto s = mk(SE::Host, v.is_int() ? Ty::Int : v.is_dbl() ? Ty::Double : Ty::Bool);
        s->host = v;
        return s;
      }
      case Atom::Int: {
        auto s = mk(SE::Const, Ty::Int);
        s->ci = a.i;
        return s;
      }
      case Atom::Double: {
        auto s = mk(SE::Const, Ty::Double);
        s->cd = a.d;
        return s;
      }
      case Atom::Bool: {
        auto s = mk(SE::Const, Ty::Bool);
        s->ci = a.b;
        return s;
      }
      case Atom::Unit: return mk(SE::Const, Ty::Unit);  // body-scope results are Unit
      default: gen_fail("non-scalar constant in a loop body");
    }
  }

  SEP sym_block(int b) {
    const Block& bl = P.blocks.at(b);
    for (int s : bl.stmts) sym_[s] = sym_stmt(P.stmts.at(s));
    return sym_atom(bl.result);
  }

  SEP sym_stmt(const Stmt& s) {
    const std::string& op = s.op;
    const Ty ty = s.ty.t;
    if (op == "Plus" || op == "Minus" || op == "Times" || op == "Divide" || op == "Lt" ||
        op == "Eq" || op == "And" || op == "Or") {
      auto e = mk(SE::Bin, ty);
      e->op = op;
      e->a = {sym_atom(s.args[0]), sym_atom(s.args[1])};
      return e;
    }
    if (op == "Not" || op == "MathAbs" || op == "MathSqrt" || op == "ToDouble" || op == "MathExp") {
      auto e = mk(SE::Un, ty);
      e->op = op;
      e->a = {sym_atom(s.args[0])};
      return e;
    }
    if (op == "IfThenElse") {
      auto c = sym_atom(s.args[0]);
      auto t = sym_block(s.blocks[0]);
      auto f = sym_block(s.blocks[1]);
      auto e = mk(SE::Sel, ty);
      e->a = {c, t, f};
      return e;
    }
    if (op == "VectorApply") {
      auto e = mk(SE::Load, ty);
      e->a = {sym_atom(s.args[0]), sym_atom(s.args[1])};
      if (e->a[0]->k != SE::Vec) gen_fail("element load from a vector produced inside the loop");
      return e;
    }
    if (op == "VectorLength") {
      auto v = sym_atom(s.args[0]);
      if (v->k != SE::Vec) gen_fail("length of a loop-local vector");
      auto e = mk(SE::Const, Ty::Int);
      e->ci = v->vec->n;
      return e;
    }
    if (op == "ParallelLoop") {
      // nested (possibly horizontally fused) loop: every live elem must be a plain reduce over
      // a loop-invariant range; each becomes one Red node bound to its elem's `out`
      const Loop& L = *s.loop;
      auto rng = sym_atom(L.range);
      int64_t range;
      if (!is_const_int(rng, &range)) gen_fail("nested reduce over a non-constant range");
      auto idx = mk(SE::Inner, Ty::Int);
      idx->sym = L.index;
      sym_[L.index] = idx;
      sym_block(L.body);
      SEP first;
      for (const Elem& e : L.elems) {
        if (!e.live) continue;
        if (e.kind != "reduce" || e.cond >= 0) gen_fail("nested loop elem other than a plain reduce");
        auto elem = sym_block(e.elem);
        sym_[e.rv_left] = mk(SE::RvL, e.out_ty.t);
        sym_[e.rv_right] = mk(SE::RvR, e.out_ty.t);
        auto comb = sym_block(e.combine);
        auto r = mk(SE::Red, e.out_ty.t);
        r->range = range;
        r->zero = e.zero;
        r->sym = L.index;
        r->a = {elem, comb};
        sym_[e.out] = r;
        if (!first) first = r;
      }
      if (!first) gen_fail("nested loop without live elems");
      return first;
    }
    gen_fail("don't know how to generate code for: " + op + " inside a multiloop");
  }

  static bool is_plus_combine(const SEP& c) {
    return c->k == SE::Bin && c->op == "Plus" &&
           ((c->a[0]->k == SE::RvL && c->a[1]->k == SE::RvR) || (c->a[0]->k == SE::RvR && c->a[1]->k == SE::RvL));
  }
  static bool is_times_combine(const SEP& c) {
    return c->k == SE::Bin && c->op == "Times" &&
           ((c->a[0]->k == SE::RvL && c->a[1]->k == SE::RvR) || (c->a[0]->k == SE::RvR && c->a[1]->k == SE::RvL));
  }

  struct LElem {
    const Elem* e;
    SEP cond, value, combine;
  };

  // ---- family: fused k-means (argmin collect + bucket counts / sums keyed on it) -----------
  struct KmeansShape {
    VecP x, mu;
    int64_t d = 0, k = 0;
  };
  // D = Red(range d, zero 0.0, Plus, Times(t, t), t = Load(X, d*Idx + J) - Load(M, c*d + J))
  bool match_distance(const SEP& D, int64_t c, KmeansShape* ks) {
    if (D->k != SE::Red || D->ty != Ty::Double || !is_plus_combine(D->a[1])) MISS("match_distance#1");
    if (D->zero.k != Atom::Double || D->zero.d != 0.0) MISS("match_distance#2");
    const SEP& el = D->a[0];
    if (el->k != SE::Bin || el->op != "Times" || !same_se(el->a[0], el->a[1])) MISS("match_distance#3");
    const SEP& t = el->a[0];
    if (t->k != SE::Bin || t->op != "Minus" || t->a[0]->k != SE::Load || t->a[1]->k != SE::Load) MISS("match_distance#4");
    auto ax = affine(t->a[0]->a[1]), am = affine(t->a[1]->a[1]);
    if (!ax || !am) MISS("match_distance#5");
    const int64_t d = D->range;
    if (ax->a != d || ax->b != 1 || ax->c != 0 || ax->inner != D->sym) MISS("match_distance#6");
    if (am->a != 0 || am->b != 1 || am->c != c * d || am->inner != D->sym) MISS("match_distance#7");
    VecP X = t->a[0]->a[0]->vec, M = t->a[1]->a[0]->vec;
    if (X->elem != Ty::Double || M->elem != Ty::Double) MISS("match_distance#8");
    if (ks->x && (ks->x != X || ks->mu != M || ks->d != d)) MISS("match_distance#9");
    ks->x = X;
    ks->mu = M;
    ks->d = d;
    return true;
  }
  // chain: idx_{c+1} = Sel(lt_c, c, idx_c), best_{c+1} = Sel(lt_c, D_c, best_c),
  // lt_c = Lt(D_c, best_c), idx_0 = 0, best_0 = 1e300 (staged_if chain, stage.cpp:73-104)
  bool match_argmin(const SEP& root, KmeansShape* ks) {
    std::vector<SEP> levels;
    SEP cur = root;
    while (cur->k == SE::Sel && cur->ty == Ty::Int) {
      levels.push_back(cur);
      cur = cur->a[2];
    }
    int64_t z;
    if (!is_const_int(cur, &z) || z != 0 || levels.empty()) MISS("match_argmin#1");
    const int64_t k = static_cast<int64_t>(levels.size());
    SEP best_prev;  // best_c
    for (int64_t c = 0; c < k; ++c) {
      const SEP& lv = levels[k - 1 - c];
      int64_t cv;
      if (!is_const_int(lv->a[1], &cv) || cv != c) MISS("match_argmin#2");
      const SEP& lt = lv->a[0];
      if (lt->k != SE::Bin || lt->op != "Lt") MISS("match_argmin#3");
      const SEP& D = lt->a[0];
      const SEP& B = lt->a[1];
      if (c == 0) {
        double bd;
        if (!is_const_dbl(B, &bd) || bd != 1e300) MISS("match_argmin#4");
      } else if (!same_se(B, best_prev)) {
        MISS("match_argmin#5");
      }
      if (!match_distance(D, c, ks)) MISS("match_argmin#6");
      // best_{c+1}: the Sel(lt, D, best_c) that the next level compares against
      auto nb = mk(SE::Sel, Ty::Double);
      nb->a = {lt, D, B};
      best_prev = nullptr;
      if (c + 1 < k) {
        const SEP& nlt = levels[k - 2 - c]->a[0];
        if (nlt->k != SE::Bin || nlt->op != "Lt") MISS("match_argmin#7");
        const SEP& nB = nlt->a[1];
        if (nB->k != SE::Sel || !same_se(nB->a[0], lt) || !same_se(nB->a[1], D) || !same_se(nB->a[2], B))
          MISS("match_argmin#8");
        best_prev = nB;
      }
    }
    ks->k = k;
    return true;
  }

  bool try_kmeans(const Loop& L, int64_t n, std::vector<LElem>& els, json& rep) {
    int ci = -1;
    for (size_t q = 0; q < els.size(); ++q)
      if (els[q].e->kind == "collect") {
        if (ci >= 0) MISS("try_kmeans#1");
        ci = static_cast<int>(q);
      }
    if (ci < 0 || els[ci].cond || els[ci].e->append) MISS("try_kmeans#2");
    KmeansShape ks;
    if (!match_argmin(els[ci].value, &ks)) MISS("try_kmeans#3");
    if (n * ks.d > ks.x->n || ks.k * ks.d > ks.mu->n) MISS("try_kmeans#4");
    const SEP key = els[ci].value;
    // reduce elems: cond Eq(key, c); value 1 (count) or Load(X, d*Idx + j) (sum)
    struct Slot { int kind; int64_t c, j; };
    std::vector<Slot> slots(els.size(), Slot{-1, 0, 0});
    for (size_t q = 0; q < els.size(); ++q) {
      if (static_cast<int>(q) == ci) continue;
      const LElem& le = els[q];
      if (le.e->kind != "reduce" || !le.cond || !is_plus_combine(le.combine)) MISS("try_kmeans#5");
      const SEP& cd = le.cond;
      if (cd->k != SE::Bin || cd->op != "Eq") MISS("try_kmeans#6");
      int64_t c;
      if (cd->a[0] == key && is_const_int(cd->a[1], &c)) {
      } else if (cd->a[1] == key && is_const_int(cd->a[0], &c)) {
      } else {
        MISS("try_kmeans#7");
      }
      if (c < 0 || c >= ks.k) MISS("try_kmeans#8");
      int64_t one;
      if (is_const_int(le.value, &one) && one == 1 && le.e->zero.k == Atom::Int && le.e->zero.i == 0) {
        slots[q] = {0, c, 0};
      } else if (le.value->k == SE::Load && le.value->a[0]->vec == ks.x && le.e->zero.k == Atom::Double &&
                 le.e->zero.d == 0.0) {
        auto af = affine(le.value->a[1]);
        if (!af || af->a != ks.d || af->b != 0 || af->c < 0 || af->c >= ks.d) MISS("try_kmeans#9");
        slots[q] = {1, c, af->c};
      } else {
        MISS("try_kmeans#10");
      }
    }
    // launch the fused multiloop kernel
    const int d = static_cast<int>(ks.d), k = static_cast<int>(ks.k);
    rep["family"] = "kmeans";
    rep["n"] = n;
    rep["d"] = d;
    rep["k"] = k;
    rep["launch"] = "dlx_kmeans_step";
    if (g_dry) return dry_bind(els), true;
    const size_t wsb = dlx_kmeans_workspace_bytes(n, d, k);
    void* ws = dalloc(wsb);
    auto* a32 = static_cast<int32_t*>(dalloc(std::max<int64_t>(1, n) * 4));
    auto* counts = static_cast<int64_t*>(dalloc(k * 8));
    auto* sums = static_cast<double*>(dalloc(static_cast<size_t>(k) * d * 8));
    int rc = dlx_kmeans_step(static_cast<const double*>(ks.x->p), n, d, k, static_cast<const double*>(ks.mu->p),
                             a32, counts, sums, ws, wsb, DLX_KMEANS_AUTO, lst_);
    VecP assign = new_vec(n, Ty::Int, lst_, false);
    if (rc == DLX_OK) rc = dlx_widen_i32_i64(a32, n, static_cast<int64_t*>(assign->p), lst_);
    int64_t* hc = res_->pin.get_n<int64_t>(k);
    double* hs = res_->pin.get_n<double>(static_cast<size_t>(k) * d);
    if (rc == DLX_OK) {
      cudaMemcpyAsync(hc, counts, k * 8, cudaMemcpyDeviceToHost, lst_);
      cudaMemcpyAsync(hs, sums, static_cast<size_t>(k) * d * 8, cudaMemcpyDeviceToHost, lst_);
    }
    dfree(ws);
    dfree(a32);
    dfree(counts);
    dfree(sums);
    ck(rc);
    std::vector<int> outs;
    std::vector<std::pair<int, int64_t>> bind;   // out sym -> index into counts (< 0: sums[~i])
    for (size_t q = 0; q < els.size(); ++q) {
      outs.push_back(els[q].e->out);
      if (static_cast<int>(q) == ci) continue;
      bind.emplace_back(els[q].e->out, slots[q].kind == 0 ? slots[q].c : ~(slots[q].c * d + slots[q].j));
    }
    defer(outs, [this, aout = els[ci].e->out, assign, hc, hs, bind = std::move(bind)] {
      env_[aout] = Val{assign};
      for (auto [o, ix] : bind) env_[o] = ix >= 0 ? Val{hc[ix]} : Val{hs[~ix]};
    });
    rep["family"] = "kmeans";
    rep["n"] = n;
    rep["d"] = d;
    rep["k"] = k;
    rep["launch"] = "dlx_kmeans_step";
    return true;
  }

  // ---- family: bucket counts (GroupBy) -------------------------------------------------------
  bool try_groupby(int64_t n, std::vector<LElem>& els, json& rep) {
    VecP keys;
    std::vector<int64_t> bucket(els.size());
    int64_t nb = 0;
    for (size_t q = 0; q < els.size(); ++q) {
      const LElem& le = els[q];
      int64_t one;
      if (le.e->kind != "reduce" || !le.cond || !is_plus_combine(le.combine) ||
          !is_const_int(le.value, &one) || one != 1 || le.e->zero.k != Atom::Int || le.e->zero.i != 0)
        return false;
      const SEP& cd = le.cond;
      if (cd->k != SE::Bin || cd->op != "Eq") return false;
      SEP ld = cd->a[0], cs = cd->a[1];
      if (ld->k != SE::Load) std::swap(ld, cs);
      int64_t b;
      if (ld->k != SE::Load || !is_const_int(cs, &b) || b < 0) return false;
      auto af = affine(ld->a[1]);
      if (!af || af->a != 1 || af->b != 0 || af->c != 0 || ld->a[0]->vec->elem != Ty::Int) return false;
      if (keys && keys != ld->a[0]->vec) return false;
      keys = ld->a[0]->vec;
      bucket[q] = b;
      nb = std::max(nb, b + 1);
    }
    if (!keys || n > keys->n || nb > (1 << 24)) return false;
    rep["family"] = "groupby";
    rep["n"] = n;
    rep["buckets"] = nb;
    rep["launch"] = "dlx_groupby_count";
    if (g_dry) return dry_bind(els), true;
    const size_t wsb = dlx_groupby_workspace_bytes(n, nb);
    void* ws = dalloc(wsb);
    auto* counts = static_cast<int64_t*>(dalloc(nb * 8));
    int rc = dlx_groupby_count(static_cast<const int64_t*>(keys->p), n, nb, counts, ws, wsb, lst_);
    int64_t* hc = res_->pin.get_n<int64_t>(nb);
    if (rc == DLX_OK) cudaMemcpyAsync(hc, counts, nb * 8, cudaMemcpyDeviceToHost, lst_);
    dfree(ws);
    dfree(counts);
    ck(rc);
    std::vector<int> outs;
    for (size_t q = 0; q < els.size(); ++q) outs.push_back(els[q].e->out);
    defer(outs, [this, outs, hc, bucket] {
      for (size_t q = 0; q < outs.size(); ++q) env_[outs[q]] = Val{hc[bucket[q]]};
    });
    rep["family"] = "groupby";
    rep["n"] = n;
    rep["buckets"] = nb;
    rep["launch"] = "dlx_groupby_count";
    return true;
  }

  // ---- family: GDA pass 2 (d*d scatter with per-class mean select) ---------------------------
  // value = Times(Minus(Load(X, d*Idx + a), Sel_a), Minus(Load(X, d*Idx + b), Sel_b)),
  // Sel = Sel(Eq(Load(Y, Idx), 1), mu1, mu0) with host scalars.
  bool match_centred(const SEP& t, VecP* X, VecP* Y, int64_t* col, double* m0, double* m1, int64_t d) {
    if (t->k != SE::Bin || t->op != "Minus" || t->a[0]->k != SE::Load || t->a[1]->k != SE::Sel) return false;
    auto af = affine(t->a[0]->a[1]);
    if (!af || af->a != d || af->b != 0 || af->c < 0 || af->c >= d) return false;
    const SEP& sel = t->a[1];
    const SEP& eq = sel->a[0];
    if (eq->k != SE::Bin || eq->op != "Eq") return false;
    SEP ld = eq->a[0], cs = eq->a[1];
    if (ld->k != SE::Load) std::swap(ld, cs);
    int64_t one;
    if (ld->k != SE::Load || !is_const_int(cs, &one) || one != 1) return false;
    auto ay = affine(ld->a[1]);
    if (!ay || ay->a != 1 || ay->b != 0 || ay->c != 0) return false;
    if (!is_const_dbl(sel->a[1], m1) || !is_const_dbl(sel->a[2], m0)) return false;
    *X = t->a[0]->a[0]->vec;
    *Y = ld->a[0]->vec;
    *col = af->c;
    return true;
  }

  bool try_gda2(int64_t n, std::vector<LElem>& els, json& rep) {
    if (els.empty()) return false;
    VecP X, Y;
    int64_t d = 0;
    // infer d from the first elem's row stride
    {
      const SEP& v = els[0].value;
      if (v->k != SE::Bin || v->op != "Times" || v->a[0]->k != SE::Bin || v->a[0]->a[0]->k != SE::Load) return false;
      auto af = affine(v->a[0]->a[0]->a[1]);
      if (!af) return false;
      d = af->a;
    }
    if (d <= 0 || d > 128) return false;
    std::vector<double> mu0(d, 0.0), mu1(d, 0.0);
    std::vector<char> seen(d, 0);
    std::vector<std::pair<int64_t, int64_t>> cell(els.size());
    for (size_t q = 0; q < els.size(); ++q) {
      const LElem& le = els[q];
      if (le.e->kind != "reduce" || le.cond || !is_plus_combine(le.combine) || le.e->zero.k != Atom::Double ||
          le.e->zero.d != 0.0)
        return false;
      const SEP& v = le.value;
      if (v->k != SE::Bin || v->op != "Times") return false;
      VecP x1, y1, x2, y2;
      int64_t a, b;
      double a0, a1, b0, b1;
      if (!match_centred(v->a[0], &x1, &y1, &a, &a0, &a1, d) || !match_centred(v->a[1], &x2, &y2, &b, &b0, &b1, d))
        return false;
      if (x1 != x2 || y1 != y2 || (X && (X != x1 || Y != y1))) return false;
      X = x1;
      Y = y1;
      for (auto [col, m0, m1] : {std::tuple{a, a0, a1}, std::tuple{b, b0, b1}}) {
        if (seen[col] && (mu0[col] != m0 || mu1[col] != m1)) return false;
        seen[col] = 1;
        mu0[col] = m0;
        mu1[col] = m1;
      }
      cell[q] = {a, b};
    }
    if (X->elem != Ty::Double || Y->elem != Ty::Int || n * d > X->n || n > Y->n) return false;
    rep["family"] = "gda_scatter";
    rep["n"] = n;
    rep["d"] = d;
    rep["launch"] = "dlx_gda_pass2";
    if (g_dry) return dry_bind(els), true;
    const size_t wsb = dlx_gda_workspace_bytes(n, static_cast<int32_t>(d));
    auto* dm0 = static_cast<double*>(dalloc(d * 8));
    auto* dm1 = static_cast<double*>(dalloc(d * 8));
    auto* S = static_cast<double*>(dalloc(d * d * 8));
    void* ws = dalloc(wsb);
    double* hmu = res_->pin.get_n<double>(2 * d);   // pinned: the copies stay asynchronous
    std::memcpy(hmu, mu0.data(), d * 8);
    std::memcpy(hmu + d, mu1.data(), d * 8);
    cudaMemcpyAsync(dm0, hmu, d * 8, cudaMemcpyHostToDevice, lst_);
    cudaMemcpyAsync(dm1, hmu + d, d * 8, cudaMemcpyHostToDevice, lst_);
    int rc = dlx_gda_pass2(static_cast<const double*>(X->p), static_cast<const int64_t*>(Y->p), n,
                           static_cast<int32_t>(d), dm0, dm1, S, ws, wsb, lst_);
    double* hS = res_->pin.get_n<double>(d * d);
    if (rc == DLX_OK) cudaMemcpyAsync(hS, S, d * d * 8, cudaMemcpyDeviceToHost, lst_);
    dfree(dm0);
    dfree(dm1);
    dfree(S);
    dfree(ws);
    ck(rc);
    std::vector<int> outs;
    std::vector<int64_t> ix;
    for (size_t q = 0; q < els.size(); ++q) {
      outs.push_back(els[q].e->out);
      ix.push_back(cell[q].first * d + cell[q].second);
    }
    defer(outs, [this, outs, ix = std::move(ix), hS] {
      for (size_t q = 0; q < outs.size(); ++q) env_[outs[q]] = Val{hS[ix[q]]};
    });
    rep["family"] = "gda_scatter";
    rep["n"] = n;
    rep["d"] = d;
    rep["launch"] = "dlx_gda_pass2";
    return true;
  }

  // ---- generic multiloop kernel (bytecode) ---------------------------------------------------------
  struct VmBuild {
    std::vector<dlx_vm_instr> code;
    std::unordered_map<const SE*, int> reg;
    std::vector<VecP> vecs;
    int nreg = 0;
  };
  int vm_emit(VmBuild& B, const SEP& s) {
    auto it = B.reg.find(s.get());
    if (it != B.reg.end()) return it->second;
    auto push = [&](uint8_t op, int a, int b, int64_t imm, int aux) {
      if (B.nreg >= DLX_VM_MAX_REGS) gen_fail("multiloop body needs more than " + std::to_string(DLX_VM_MAX_REGS) + " registers");
      dlx_vm_instr in{};
      in.op = op;
      in.dst = static_cast<uint8_t>(B.nreg);
      in.a = static_cast<uint8_t>(a);
      in.b = static_cast<uint8_t>(b);
      in.imm = imm;
      in.aux = aux;
      B.code.push_back(in);
      return B.nreg++;
    };
    int r = -1;
    switch (s->k) {
      case SE::Const: {
        int64_t bits = s->ci;
        if (s->ty == Ty::Double) std::memcpy(&bits, &s->cd, 8);
        r = push(DLX_VM_CONST, 0, 0, bits, 0);
        break;
      }
      case SE::Host: {
        int64_t bits = 0;
        if (s->host.is_int()) bits = s->host.i();
        else if (s->host.is_dbl()) { double dv = s->host.d(); std::memcpy(&bits, &dv, 8); }
        else if (s->host.is_bool()) bits = s->host.b();
        else gen_fail("non-scalar host value in a loop body");
        r = push(DLX_VM_CONST, 0, 0, bits, 0);
        break;
      }
      case SE::Idx: r = push(DLX_VM_IDX, 0, 0, 0, 0); break;
      case SE::Load: {
        const VecP& v = s->a[0]->vec;
        int vi = -1;
        for (size_t q = 0; q < B.vecs.size(); ++q)
          if (B.vecs[q] == v) vi = static_cast<int>(q);
        if (vi < 0) {
          if (B.vecs.size() >= DLX_VM_MAX_VECS) gen_fail("multiloop reads too many vectors");
          vi = static_cast<int>(B.vecs.size());
          B.vecs.push_back(v);
        }
        const int ir = vm_emit(B, s->a[1]);
        r = push(DLX_VM_LOAD, ir, 0, 0, vi);
        break;
      }
      case SE::Bin: {
        const int x = vm_emit(B, s->a[0]), y = vm_emit(B, s->a[1]);
        const bool dbl = s->a[0]->ty == Ty::Double;
        const std::string& op = s->op;
        uint8_t o;
        if (op == "Plus") o = dbl ? DLX_VM_ADD_D : DLX_VM_ADD_I;
        else if (op == "Minus") o = dbl ? DLX_VM_SUB_D : DLX_VM_SUB_I;
        else if (op == "Times") o = dbl ? DLX_VM_MUL_D : DLX_VM_MUL_I;
        else if (op == "Divide") o = dbl ? DLX_VM_DIV_D : DLX_VM_DIV_I;
        else if (op == "Lt") o = dbl ? DLX_VM_LT_D : DLX_VM_LT_I;
        else if (op == "Eq") o = dbl ? DLX_VM_EQ_D : DLX_VM_EQ_I;
        else if (op == "And") o = DLX_VM_AND;
        else if (op == "Or") o = DLX_VM_OR;
        else gen_fail("operator " + op);
        r = push(o, x, y, 0, 0);
        break;
      }
      case SE::Un: {
        const int x = vm_emit(B, s->a[0]);
        const std::string& op = s->op;
        uint8_t o;
        if (op == "Not") o = DLX_VM_NOT;
        else if (op == "MathAbs") o = s->ty == Ty::Double ? DLX_VM_ABS_D : DLX_VM_ABS_I;
        else if (op == "MathSqrt") o = DLX_VM_SQRT;
        else if (op == "MathExp") o = DLX_VM_EXP;
        else if (op == "ToDouble") o = DLX_VM_TODBL;
        else gen_fail("operator " + op);
        r = push(o, x, 0, 0, 0);
        break;
      }
      case SE::Sel: {
        const int c = vm_emit(B, s->a[0]), t = vm_emit(B, s->a[1]), f = vm_emit(B, s->a[2]);
        r = push(DLX_VM_SEL, t, f, c, 0);
        break;
      }
      default: gen_fail("nested reduce in a generic multiloop");
    }
    B.reg[s.get()] = r;
    return r;
  }

  static int vm_ty(Ty t) { return t == Ty::Double ? DLX_VM_F64 : t == Ty::Bool ? DLX_VM_BOOL : DLX_VM_I64; }

  bool run_vm(int64_t n, std::vector<LElem>& els, json& rep) {
    if (els.size() > DLX_VM_MAX_ELEMS) gen_fail("multiloop with more than 16 live elems outside the specialised families");
    VmBuild B;
    dlx_vm_loop L{};
    L.range = n;
    L.body_end = 0;
    L.nelems = static_cast<int>(els.size());
    std::vector<VecP> outs(els.size());
    for (size_t q = 0; q < els.size(); ++q) {
      const LElem& le = els[q];
      dlx_vm_elem& ve = L.elem[q];
      if (le.e->kind == "collect") {
        // filter-collect (append): order-preserving compaction, length returned in d_results
        ve.kind = le.e->append ? DLX_VM_APPEND : DLX_VM_COLLECT;
        ve.ty = vm_ty(le.e->out_ty.elem);
        outs[q] = new_vec(n, le.e->out_ty.elem == Ty::Double ? Ty::Double : le.e->out_ty.elem == Ty::Bool ? Ty::Bool : Ty::Int,
                          lst_, true);
        ve.out = outs[q]->p;
      } else if (le.e->kind == "reduce") {
        ve.kind = DLX_VM_REDUCE;
        ve.ty = vm_ty(le.e->out_ty.t);
        if (is_plus_combine(le.combine)) ve.combine = DLX_VM_COMBINE_ADD;
        else if (is_times_combine(le.combine)) ve.combine = DLX_VM_COMBINE_MUL;
        else gen_fail("reduce combine other than + or *");
        int64_t bits = le.e->zero.i;
        if (le.e->zero.k == Atom::Double) std::memcpy(&bits, &le.e->zero.d, 8);
        ve.zero = bits;
      } else {
        gen_fail("foreach elems are not lowered (disjoint-write contract, SPEC.md:673)");
      }
      // each elem gets its own code ranges; shared sub-DAGs are re-emitted per elem so a
      // guarded elem never reads a register computed under another elem's guard
      B.reg.clear();
      if (le.cond) {
        ve.cond_begin = static_cast<int>(B.code.size());
        ve.cond_reg = vm_emit(B, le.cond);
        ve.cond_end = static_cast<int>(B.code.size());
      } else {
        ve.cond_begin = ve.cond_end = static_cast<int>(B.code.size());
      }
      ve.value_begin = static_cast<int>(B.code.size());
      ve.value_reg = vm_emit(B, le.value);
      ve.value_end = static_cast<int>(B.code.size());
      B.nreg = 0;  // registers are reused per elem
    }
    if (B.code.size() > DLX_VM_MAX_CODE) gen_fail("multiloop body too large for the generic kernel");
    L.ncode = static_cast<int>(B.code.size());
    L.nvecs = static_cast<int>(B.vecs.size());
    for (size_t q = 0; q < B.vecs.size(); ++q) {
      L.vec[q] = B.vecs[q]->p;
      L.vec_len[q] = B.vecs[q]->n;
      L.vec_kind[q] = vm_ty(B.vecs[q]->elem);
    }
    rep["family"] = "generic";
    rep["n"] = n;
    rep["elems"] = static_cast<int>(els.size());
    rep["instructions"] = static_cast<int>(B.code.size());
    rep["launch"] = "dlx_vm_run_loop";
    if (g_dry) return dry_bind(els), true;
    const size_t wsb = dlx_vm_workspace_bytes(n);
    const size_t code_bytes = std::max<size_t>(1, B.code.size()) * sizeof(dlx_vm_instr);
    auto* dcode = static_cast<dlx_vm_instr*>(dalloc(code_bytes));
    auto* dres = static_cast<int64_t*>(dalloc((DLX_VM_MAX_ELEMS + 1) * 8));   // results, then the trap word
    int* dtrap = reinterpret_cast<int*>(dres + DLX_VM_MAX_ELEMS);
    void* ws = dalloc(wsb);
    // staged through pinned memory so the copies (and the launch) do not block the host
    auto* hin = res_->pin.get_n<unsigned char>(code_bytes + (DLX_VM_MAX_ELEMS + 1) * 8);
    if (!B.code.empty()) std::memcpy(hin, B.code.data(), B.code.size() * sizeof(dlx_vm_instr));
    auto* zeros = reinterpret_cast<int64_t*>(hin + ((code_bytes + 7) & ~size_t{7}));
    std::memset(zeros, 0, (DLX_VM_MAX_ELEMS + 1) * 8);
    for (size_t q = 0; q < els.size(); ++q) zeros[q] = L.elem[q].zero;
    cudaMemcpyAsync(dcode, hin, B.code.size() * sizeof(dlx_vm_instr), cudaMemcpyHostToDevice, lst_);
    cudaMemcpyAsync(dres, zeros, (DLX_VM_MAX_ELEMS + 1) * 8, cudaMemcpyHostToDevice, lst_);
    int rc = dlx_vm_run_loop(dcode, &L, dres, dtrap, ws, wsb, lst_);
    int64_t* res = res_->pin.get_n<int64_t>(DLX_VM_MAX_ELEMS + 1);
    if (rc == DLX_OK) cudaMemcpyAsync(res, dres, (DLX_VM_MAX_ELEMS + 1) * 8, cudaMemcpyDeviceToHost, lst_);
    dfree(dcode);
    dfree(dres);
    dfree(ws);
    ck(rc);
    std::vector<int> out_syms;
    std::vector<const Elem*> es;
    for (const LElem& le : els) {
      out_syms.push_back(le.e->out);
      es.push_back(le.e);
    }
    defer(out_syms, [this, res, es = std::move(es), outs = std::move(outs)] {
      int htrap;
      std::memcpy(&htrap, res + DLX_VM_MAX_ELEMS, sizeof(int));
      if (htrap & 1) trap("TrapDivByZero: integer division by zero in a multiloop");
      if (htrap & 2) trap("TrapIndexOutOfBounds: element load out of range in a multiloop");
      if (htrap & 4) gen_fail("generic kernel met an unknown instruction");
      for (size_t q = 0; q < es.size(); ++q) {
        const Elem& e = *es[q];
        if (e.kind == "collect") {
          if (e.append) outs[q]->n = res[q];   // the builder's final length
          env_[e.out] = Val{outs[q]};
        } else if (e.out_ty.t == Ty::Double) {
          double dv;
          std::memcpy(&dv, &res[q], 8);
          env_[e.out] = Val{dv};
        } else if (e.out_ty.t == Ty::Bool) {
          env_[e.out] = Val{res[q] != 0};
        } else {
          env_[e.out] = Val{res[q]};
        }
      }
    });
    rep["family"] = "generic";
    rep["n"] = n;
    rep["elems"] = static_cast<int>(els.size());
    rep["instructions"] = static_cast<int>(B.code.size());
    rep["launch"] = "dlx_vm_run_loop";
    return true;
  }

  void dry_bind(const std::vector<LElem>& els) {
    for (const LElem& le : els) {
      if (le.e->kind == "collect") env_[le.e->out] = Val{new_vec(dry_n_, le.e->out_ty.elem, st_, false)};
      else if (le.e->out_ty.t == Ty::Double) env_[le.e->out] = Val{1.0};
      else if (le.e->out_ty.t == Ty::Bool) env_[le.e->out] = Val{false};
      else env_[le.e->out] = Val{int64_t{1}};
    }
  }

  // ---- one root ParallelLoop -------------------------------------------------------------------
  Val run_loop(const Stmt& s) {
    if (g_dry) return run_loop_impl(s);
    flush_mirrors();
    // next loop stream, ordered after everything the main stream has enqueued so far (RNG
    // fills, literals, mirror flushes: the loop's inputs)
    lst_ = res_->loop[launches_++ % kLoopStreams];
    cudaEvent_t ev = get_event();
    ckc(cudaEventRecord(ev, st_), "cudaEventRecord");
    ckc(cudaStreamWaitEvent(lst_, ev, 0), "cudaStreamWaitEvent");
    res_->events.push_back(ev);
    const size_t inflight = pending_.size();
    Val r = run_loop_impl(s);
    if (!report.empty() && report.back().contains("launch")) {
      report.back()["stream"] = static_cast<int>((launches_ - 1) % kLoopStreams);
      report.back()["in_flight"] = static_cast<int>(inflight);   // loops it may overlap
    }
    invalidate_mirrors();
    return r;
  }

  Val run_loop_impl(const Stmt& s) {
    const Loop& L = *s.loop;
    const int64_t n = atom(L.range).i();
    dry_n_ = n;
    loop_index_ = L.index;
    sym_.clear();
    sym_block(L.body);
    std::vector<LElem> els;
    for (const Elem& e : L.elems) {
      if (!e.live) continue;
      LElem le{&e, nullptr, nullptr, nullptr};
      if (e.cond >= 0) le.cond = sym_block(e.cond);
      le.value = sym_block(e.elem);
      if (e.kind == "reduce") {
        sym_[e.rv_left] = mk(SE::RvL, e.out_ty.t);
        sym_[e.rv_right] = mk(SE::RvR, e.out_ty.t);
        le.combine = sym_block(e.combine);
      }
      els.push_back(le);
    }
    json rep;
    rep["loop"] = "x" + std::to_string(s.sym);
    rep["live_elems"] = static_cast<int>(els.size());
    bool done = false;
    if (n == 0) {
      for (const LElem& le : els) {
        if (le.e->kind == "collect") env_[le.e->out] = Val{new_vec(0, le.e->out_ty.elem, st_, true)};
        else env_[le.e->out] = atom(le.e->zero);
      }
      rep["family"] = "empty";
      done = true;
    }
    if (!done) done = try_kmeans(L, n, els, rep);
    if (!done) done = try_groupby(n, els, rep);
    if (!done) done = try_gda2(n, els, rep);
    if (!done) done = run_vm(n, els, rep);
    report.push_back(rep);
    loop_index_ = -1;
    sym_.clear();
    return Val{};
  }
};

}  // namespace

// Parsed descriptors by content: a caller that runs the same staged program again (an
// iteration driver, a benchmark, a server) skips the JSON parse, which dominates the host time
// of large programs (a k = 8, d = 16 k-means iteration is ~1 MB of descriptor).
std::shared_ptr<const Program> cached_program(const std::string& text) {
  static std::mutex mu;
  static std::unordered_map<std::string, std::shared_ptr<const Program>> cache;
  static std::vector<std::string> order;   // FIFO eviction, a handful of programs
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(text);
    if (it != cache.end()) return it->second;
  }
  auto p = std::make_shared<const Program>(parse_program(text));
  std::lock_guard<std::mutex> lk(mu);
  if (cache.emplace(text, p).second) {
    order.push_back(text);
    if (order.size() > 8) {
      cache.erase(order.front());
      order.erase(order.begin());
    }
  }
  return p;
}

RunResult run_program(const std::string& program_json, uint64_t seed, int device) {
  g_dry = getenv("DLX_PROGRAM_DRYRUN") != nullptr;
  g_debug = getenv("DLX_PROGRAM_DEBUG") != nullptr;
  g_no_mirror = getenv("DLX_PROGRAM_NO_MIRROR") != nullptr;
  g_serial = getenv("DLX_PROGRAM_SERIAL") != nullptr;
  const std::shared_ptr<const Program> pp = cached_program(program_json);
  const Program& p = *pp;
  cudaStream_t st = nullptr;
  if (!g_dry) {
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) throw std::runtime_error(std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
      throw std::runtime_error("cudaStreamCreate failed");
  }
  RunResult r;
  try {
    Executor ex(p, seed, st, g_dry ? nullptr : &device_res(device));
    struct VecRegistry {   // route new_vec registrations / frees to this run's executor
      VecRegistry(std::vector<std::weak_ptr<DevVec>>* r, std::function<void()>* f, cudaStream_t s) {
        g_vecs = r;
        g_fence = f;
        g_main_st = s;
      }
      ~VecRegistry() {
        g_vecs = nullptr;
        g_fence = nullptr;
      }
    } reg(&ex.vecs_, g_dry ? nullptr : &ex.fence_, st);
    Val v = ex.run();
    if (!g_dry) cudaStreamSynchronize(st);
    r.output = ex.output;
    r.result = format_val(v);
    r.report = ex.report.dump();
  } catch (const Fail& f) {
    if (!g_dry) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
    if (f.code == DLX_ERR_GENERATION) throw GenerationFailed(f.what());
    if (f.code == DLX_ERR_TRAP) throw TrapError(f.what());
    throw std::runtime_error(f.what());
  }
  if (!g_dry) cudaStreamDestroy(st);
  return r;
}

}  // namespace dlx

extern "C" {

int dlx_program_run(const char* program_json, uint64_t seed, int device, char** out_text,
                    char** out_report) {
  if (!program_json || !out_text) {
    dlx::set_error("dlx_program_run: null argument");
    return DLX_ERR_ARG;
  }
  try {
    dlx::RunResult r = dlx::run_program(program_json, seed, device);
    *out_text = strdup(r.output.c_str());
    if (out_report) *out_report = strdup(r.report.c_str());
    return DLX_OK;
  } catch (const dlx::GenerationFailed& e) {
    dlx::set_error("%s", e.what());
    return DLX_ERR_GENERATION;
  } catch (const dlx::TrapError& e) {
    dlx::set_error("%s", e.what());
    return DLX_ERR_TRAP;
  } catch (const nlohmann::json::exception& e) {
    dlx::set_error("dlx_program_run: malformed descriptor: %s", e.what());
    return DLX_ERR_ARG;
  } catch (const std::exception& e) {
    dlx::set_error("%s", e.what());
    return DLX_ERR_CUDA;
  }
}

void dlx_string_free(char* s) { free(s); }

}  // extern "C"
