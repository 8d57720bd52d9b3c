// program_exec.hpp — the executor's runtime types (device vectors, lazy loop results, values),
// the cached loop lowering (LoopPlan) and the Executor class.  program.cpp implements the host
// interpretation and the API; lower.cpp the symbolic evaluation of loop bodies, the family
// matchers and the launches.
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <functional>
#include <map>
#include <deque>
#include <memory>
#include <string>
#include <variant>
#include <vector>

#include <json.hpp>

#include "../../include/dlx.h"
#include "../../include/dlx_program.h"
#include "../../include/dlx_vm.h"
#include "jit.hpp"
#include "program_ir.hpp"

namespace dlx {

void set_error(const char* fmt, ...);
void ckc(cudaError_t e, const char* what);
void ck(int rc);

using ExecOpts = dlx_exec_options;

// one execution's context (thread-local: a thread runs one program at a time)
struct RunCtx {
  bool dry = false;      // DLX_EXEC_DRYRUN: no device work; loops are lowered and reported
  bool debug = false;    // DLX_PROGRAM_DEBUG=1: why a specialised family did not match
  bool serial = false;   // complete every loop before the next statement
  bool nocache = false;
  bool profile = false;  // DLX_PROGRAM_PROFILE=1: host time of launches, joins and the run
  cudaStream_t main = nullptr;
  std::function<void()>* fence = nullptr;
  std::chrono::steady_clock::time_point t0;   // run start (profile timestamps)
  double ms() const { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); }
};
extern thread_local RunCtx* g_run;

constexpr size_t kMirrorBytes = 64 << 10;
constexpr int64_t kPageElems = 8192;   // read-through page of a large vector (64 KiB of fp64)
constexpr int kLoopStreams = 4;

// Device vector (DenseVector mirror of VecData, runtime.hpp:44-72).
struct DevVec {
  void* p = nullptr;
  int64_t n = 0;
  Ty elem = Ty::Double;
  bool i32 = false;        // an Int vector stored as int32 on the device (k-means assignments)
  bool borrowed = false;   // the caller's device buffer (dlx_program_input.d_data): never freed
  cudaStream_t fst = nullptr;   // stream the buffer is freed on (stream-ordered allocator)
  cudaEvent_t wev = nullptr;    // a loop-stream write not yet joined (readers wait on it)
  std::vector<unsigned char> host;   // host mirror (small vectors), reference layout
  bool host_valid = false;
  std::vector<unsigned char> page;   // read-through page (large vectors), device layout
  int64_t page_lo = 0;
  bool page_valid = false;
  int64_t dirty_lo = INT64_MAX, dirty_hi = -1;   // [lo, hi) newer on the host than on the device
  // small vectors a loop is still writing: one asynchronous copy of the whole vector into pinned
  // staging serves every printed element read until the next join (device layout)
  const unsigned char* snap = nullptr;
  cudaEvent_t snap_of = nullptr;   // the write (wev) the snapshot follows
  // a synthetic source (VectorRand / VectorRandInt, not written since): shard windows on other
  // devices are drawn there by skip-ahead (shard.cpp)
  bool gen = false, gen_int = false;
  uint64_t gen_seed = 0, gen_first = 0;
  int64_t gen_bound = 0;
  uint64_t ver = 0;   // bumped by every write (host stores, copy runs, device update groups, widening)
  struct Win {        // elements [lo, hi) on a shard's device (shard.cpp)
    int shard = -1, dev = -1;
    void* p = nullptr;
    int64_t lo = 0, hi = 0;
    uint64_t ver = 0;
    cudaStream_t st = nullptr;
  };
  std::vector<Win> wins;
  void touched() {
    ++ver;
    gen = false;
  }
  ~DevVec();
  size_t esize() const { return elem == Ty::Bool ? 1 : i32 ? 4 : 8; }   // device element bytes
  size_t hsize() const { return elem == Ty::Bool ? 1 : 8; }            // host element bytes
  bool mirrored() const { return static_cast<size_t>(n) * hsize() <= kMirrorBytes; }
};
using VecP = std::shared_ptr<DevVec>;

// A scalar loop result still on its way back (its bits arrive in pinned staging when the loop
// completes; `ready` once copied out at a join).
struct Lazy {
  const unsigned char* src = nullptr;
  int64_t bits = 0;
  Ty ty = Ty::Int;
  int esz = 8;
  bool ready = false;
};
using LazyP = Lazy*;   // owned by the run's Executor (lazies_), which outlives every Val of the run

struct Cell;
using CellP = std::shared_ptr<Cell>;
struct Val {
  std::variant<std::monostate, int64_t, double, bool, std::string, VecP, CellP, LazyP> v;
  bool is_int() const { return std::holds_alternative<int64_t>(v); }
  bool is_dbl() const { return std::holds_alternative<double>(v); }
  bool is_bool() const { return std::holds_alternative<bool>(v); }
  bool is_vec() const { return std::holds_alternative<VecP>(v); }
  bool is_lazy() const { return std::holds_alternative<LazyP>(v); }
  int64_t i() const { return std::get<int64_t>(v); }
  double d() const { return std::get<double>(v); }
  bool b() const { return std::get<bool>(v); }
  const VecP& vec() const { return std::get<VecP>(v); }
};
struct Cell {
  Val v;
};
std::string format_val(const Val& x);

struct PinnedArena {
  std::vector<std::pair<unsigned char*, size_t>> blocks;   // the last block is the current one
  size_t used = 0;
  void* get(size_t bytes);
  template <class T>
  T* get_n(size_t n) { return static_cast<T*>(get(n * sizeof(T))); }
  void reset();
};
struct DeviceRes {
  cudaStream_t main = nullptr;   // host statements, RNG fills, uploads, frees
  cudaStream_t loop[kLoopStreams] = {};
  std::vector<cudaEvent_t> events;   // free list
  PinnedArena pin;
  bool init = false;
};
DeviceRes& device_res(int device);

// ---- symbolic expressions of loop bodies (lower.cpp) ------------------------------------------
struct SE;
using SEP = std::shared_ptr<SE>;
struct SE {
  enum K { Const, Idx, Inner, Host, Vec, Load, Bin, Un, Sel, Red, RvL, RvR } k;
  Ty ty = Ty::Int;
  Op op = Op::Unknown;
  int64_t ci = 0;
  double cd = 0;
  Val host;
  VecP vec;
  int sym = -1;            // Host / Vec: the env symbol; Inner / Red: the inner index symbol
  std::vector<SEP> a;      // children (Red: elem, combine)
  int64_t range = 0;       // Red
  Atom zero;               // Red
};

// A lowered root loop, cached per loop statement in the Program (valid while the inputs it
// was matched against keep their element types and lengths and every baked host scalar its
// value).
struct LoopPlan {
  enum Fam { Kmeans, GroupBy, BucketRows, GdaScatter, Logistic, Generic, Compiled } fam = Generic;
  std::string family, launch;
  // inputs: env symbols of the vectors the loop reads (slot order), their types and lengths
  std::vector<int> vsyms;
  std::vector<Ty> vtys;
  std::vector<int64_t> vlens;
  std::vector<std::pair<int, int64_t>> baked;   // host scalars structural to the match
  std::vector<int> deps;                        // every env symbol the body reads
  int64_t d = 0, k = 0;                         // k-means d, k; bucket rows d, K; GDA d; GroupBy K
  int x = -1, mu = -1, keys = -1;               // input slots
  // outputs: per live elem, the symbol and where its value comes from
  struct Out {
    int sym;
    int src;        // 0: scalar slot ix of the staged result record; 1: the collect vector
    int64_t ix;
    Ty ty;
    bool group_only = false;   // read only by the update group (not copied back when it is fused)
  };
  std::vector<Out> outs;
  int64_t nres = 0;                             // 64-bit slots in the staged result record
  // k-means: the update group run on the device
  int upd_vec = -1;                             // V's symbol (-1: none)
  std::vector<int> skip;                        // the group's host statements
  bool sums_group_only = false;                 // every sum is read only by the group
  // logistic: the link expression of the dot (host scalars re-read per launch) and the axpy
  // update group's alpha (a literal, or a host symbol)
  dlx_link_code link{};
  std::vector<std::pair<int, int>> link_patches;   // (instruction, host symbol)
  int alpha_sym = -1;
  double alpha_lit = 0;
  // bucket counts / bucket rows: bucket values
  std::vector<int64_t> buckets;
  // GDA scatter: per column the class-mean sources (symbol, or -1 and a literal)
  std::vector<int> m0sym, m1sym;
  std::vector<double> m0lit, m1lit;
  std::vector<int64_t> cell;                    // per elem a*d + b
  // generic kernel
  std::vector<dlx_vm_instr> code;
  dlx_vm_loop L{};
  std::vector<std::pair<int, int>> patches;     // (instruction, host symbol): constants re-read per launch
  std::vector<Ty> coll_ty;                      // per elem collect element type
  // compiled (NVRTC) kernel of the loop body (lower_jit.cpp)
  std::string jit_src;
  std::vector<std::string> jit_names;
  std::vector<uint8_t> jit_kind;                // per elem: 0 reduce, 1 collect, 2 append
  std::vector<int> jit_host;                    // host scalars read per launch (env symbols)
  int jit_nred = 0, jit_napp = 0, jit_words = 0;
  std::shared_ptr<const JitModule> jit;         // compiled on first launch (process-wide cache)
};

struct MatchCtx {   // what a lowering depends on (recorded into the LoopPlan)
  std::vector<int> vsyms;
  std::vector<VecP> vecs;
  std::vector<std::pair<int, int64_t>> baked;
  std::vector<int> deps;
  int slot(const SEP& vn);
  void bake(const SEP& s);
};

// A per-symbol environment (values, bound / skip flags), pooled in the Program across runs;
// `touched` lists the symbols to clear when it goes back.
struct Scratch {
  std::vector<Val> env;
  std::vector<uint8_t> bound, skip;
  std::vector<int> touched;
};

// ---- the executor ----------------------------------------------------------------------------
class Executor {
 public:
  Executor(const Program& p, const ExecOpts& o, cudaStream_t st, DeviceRes* res);
  ~Executor();
  Val run();
  std::string output() const;
  Val force(Val v);
  void join_all();
  void widen(const VecP& v, cudaStream_t s);
  nlohmann::json report = nlohmann::json::array();
  std::function<void()> fence_;   // RunCtx::fence points here during the run
  // one contiguous index shard of a sharded loop (shard.cpp)
  struct Shard {
    int g = 0, dev = 0;
    int64_t lo = 0, hi = 0;
    cudaStream_t st = nullptr;
    bool local = true;   // on the primary device, reading the vectors in place
  };

 private:
  const Program& P;
  ExecOpts opts_;
  std::vector<int> devs_;     // ExecOptions.devices; devs_[0] is the primary (vectors live there)
  int primary_ = 0;
  bool replicate_ = false;    // DLX_SHARD_REPLICATE=1: shard windows even on the primary (tests)
  std::vector<std::pair<int, cudaEvent_t>> xevents_;   // events created on shard devices
  uint64_t draws_ = 0;
  cudaStream_t st_;
  DeviceRes* res_;
  cudaStream_t lst_;   // stream of the loop being launched
  int64_t launches_ = 0;
  std::shared_ptr<Scratch> sc_;
  std::vector<Val>& env_;
  std::vector<uint8_t>& bound_;
  std::vector<uint8_t>& skip_;
  std::vector<std::weak_ptr<DevVec>> vecs_;   // every vector of this run
  std::vector<std::string> lines_;            // printed output
  std::vector<std::pair<size_t, LazyP>> prints_;   // lines waiting for a loop result
  std::vector<LazyP> unresolved_;
  std::deque<Lazy> lazies_;   // every lazy of this run (stable addresses; no refcounting per bind)
  bool main_async_ = false;                   // main-stream work reads pinned staging
  cudaEvent_t prof_t0_ = nullptr;             // DLX_PROGRAM_PROFILE: run start on the main stream

  struct Pending {
    cudaEvent_t ev;                 // recorded on the loop's stream after its result copies
    std::function<void()> finish;   // binds deferred outputs / raises the loop's traps
  };
  std::vector<Pending> pending_;   // launch (= program) order

  cudaEvent_t get_event();
  cudaEvent_t complete_loop(const std::vector<int>& deferred_outs, std::function<void()> fn);
  void fence();
  void fence_on(cudaStream_t s);
  static Val lazy_val(const Lazy& l);
  void format_prints();   // the deferred prints of joined loops (parallel on a host pool)
  LazyP make_lazy(const void* src, Ty ty, int esz);
  void bind(int sym, Val v) {
    env_[sym] = std::move(v);
    if (!bound_[sym]) sc_->touched.push_back(sym);
    bound_[sym] = 1;
  }
  void mark_skip(int sym) {
    skip_[sym] = 1;
    sc_->touched.push_back(sym);
  }

  Val atomv(const Atom& a);                     // may be a Lazy
  Val atom(const Atom& a) { return force(atomv(a)); }
  VecP vec_of(const Atom& a);
  VecP new_vec(int64_t n, Ty elem, cudaStream_t st, bool zero, bool i32 = false);
  void load_mirror(const VecP& v);
  void flush_mirrors();
  static Val host_elem(const unsigned char* h, Ty elem);
  Val vec_get(const VecP& v, int64_t i);
  void vec_set(const VecP& v, int64_t i, const Val& x);
  Val exec_block(int b);
  bool copy_run(const CopyRun& run);
  Val exec_stmt(const Stmt& s);
  Val scalar(Op op, const Val& x, const Val& y);

  // ---- loops (lower.cpp) ----
  int loop_index_ = -1;
  int64_t dry_n_ = 0;
  std::unordered_map<int, SEP> sym_;
  MatchCtx* mc_ = nullptr;
  struct LElem {
    const Elem* e;
    SEP cond, value, combine;
  };
  void run_loop(const Stmt& s);
  std::shared_ptr<LoopPlan> lower(const Stmt& s, int64_t n);
  bool plan_valid(const LoopPlan& p, std::vector<VecP>& vecs);
  void launch(const Stmt& s, LoopPlan& p, int64_t n, std::vector<VecP>& vecs, nlohmann::json& rep);
  void bind_empty(const Loop& L);
  SEP sym_atom(const Atom& a);
  SEP sym_block(int b);
  SEP sym_stmt(const Stmt& s);
  bool is_const_int(const SEP& s, int64_t* v = nullptr);
  bool is_const_dbl(const SEP& s, double* v = nullptr);
  struct Affine {
    int64_t a = 0, b = 0, c = 0;
    int inner = -1;
  };
  bool affine(const SEP& s, Affine* out);
  // family matchers: fill the plan and return true, or return false (not this family)
  bool match_distance(const SEP& D, int64_t c, LoopPlan& p, MatchCtx& m);
  bool match_argmin(const SEP& root, LoopPlan& p, MatchCtx& m);
  bool match_kmeans(const Stmt& s, int64_t n, std::vector<LElem>& els, LoopPlan& p, MatchCtx& m);
  bool match_groupby(int64_t n, std::vector<LElem>& els, LoopPlan& p, MatchCtx& m);
  bool match_bucket_rows(int64_t n, std::vector<LElem>& els, LoopPlan& p, MatchCtx& m);
  bool match_centred(const SEP& t, int64_t d, int* xs, int* ys, int64_t* col, int* s0, double* l0, int* s1, double* l1,
                     MatchCtx& m);
  bool match_gda2(int64_t n, std::vector<LElem>& els, LoopPlan& p, MatchCtx& m);
  bool match_logistic(const Stmt& s, int64_t n, std::vector<LElem>& els, LoopPlan& p, MatchCtx& m);
  bool link_compile(const SEP& f, const SEP& dot, LoopPlan& p, std::unordered_map<const SE*, int>& reg);
  bool match_generic(int64_t n, std::vector<LElem>& els, LoopPlan& p, MatchCtx& m);
  bool match_compiled(int64_t n, std::vector<LElem>& els, LoopPlan& p, MatchCtx& m);
  int vm_emit(LoopPlan& p, MatchCtx& m, std::unordered_map<const SE*, int>& reg, int& nreg, const SEP& s);
  // launches
  void launch_kmeans(const Stmt& s, LoopPlan& p, int64_t n, std::vector<VecP>& V, nlohmann::json& rep);
  void launch_groupby(LoopPlan& p, int64_t n, std::vector<VecP>& V);
  void launch_bucket_rows(LoopPlan& p, int64_t n, std::vector<VecP>& V);
  void launch_gda2(LoopPlan& p, int64_t n, std::vector<VecP>& V);
  void launch_logistic(LoopPlan& p, int64_t n, std::vector<VecP>& V, nlohmann::json& rep);
  void launch_generic(LoopPlan& p, int64_t n, std::vector<VecP>& V);
  void launch_compiled(LoopPlan& p, int64_t n, std::vector<VecP>& V);
  // sharded launches (shard.cpp)
  bool sharded(const LoopPlan& p) const;
  std::vector<Shard> shards(int64_t n);
  cudaEvent_t dev_event(int dev);
  const void* window(const VecP& v, const Shard& s, int64_t lo, int64_t hi);
  void run_shards(std::vector<Shard>& sh, const std::function<void(Shard&)>& body);
  void launch_kmeans_sharded(LoopPlan& p, int64_t n, std::vector<VecP>& V, nlohmann::json& rep);
  void launch_groupby_sharded(LoopPlan& p, int64_t n, std::vector<VecP>& V);
  void launch_bucket_rows_sharded(LoopPlan& p, int64_t n, std::vector<VecP>& V);
  void launch_gda2_sharded(LoopPlan& p, int64_t n, std::vector<VecP>& V);
  void launch_logistic_sharded(LoopPlan& p, int64_t n, std::vector<VecP>& V, nlohmann::json& rep);
  void bind_scalars(const LoopPlan& p, const int64_t* hres);
  void* dalloc(size_t bytes);
  void dfree(void* p);
  void wait_inputs(const std::vector<VecP>& V);
};

}  // namespace dlx
