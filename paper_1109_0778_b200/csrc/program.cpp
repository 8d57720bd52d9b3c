// program.cpp — the multiloop program executor: the B200 replacement for the reference's
// missing interpret() / executeDEG() (interp.hpp:10).  See
// include/dlx_program.h for the contract and include/dlx/executor.hpp for the C++ API.
//
// Execution model (mirrors SPEC.md's runtime module):
//   * root-block statements run in schedule order; single-task scalar statements (the Op set
//     of node.hpp:14-48, IfThenElse, While, Var*) on the host with the reference semantics:
//     Int wraps (graph.cpp:10-21), Int division by zero traps, Double is IEEE;
//   * vectors are device-resident (DenseVector mirrors of VecData, runtime.hpp:44-72);
//     VectorRand / VectorRandInt draw from one Rng(seed) in program order on the device, or take
//     caller-supplied data (dlx_program_input);
//   * every ParallelLoop (LoopPayload, node.hpp:76-81) is lowered by the CUDA target (lower.cpp:
//     symbolic evaluation of its live elems, then the specialised families — fused k-means,
//     bucket counts, bucket row sums, GDA scatter — or the generic multiloop kernel).  The
//     lowering is cached per loop statement in the program handle;
//   * scheduleDEG's concurrency: loops run on loop streams; their results
//     stay on the device and come back asynchronously.  A data edge to a later loop is a
//     device-side event wait; a data edge to the host is a lazy value that is only waited for
//     when the host needs it (a Print of a pending result is filled in when it arrives).  So the
//     host runs ahead of the device, e.g. the k-means iterations of a staged program are all
//     enqueued back to back, each iteration's centroid update (k*d host statements in the
//     reference) executed on the device in the loop's combine launch.
#include "program_exec.hpp"

#include <algorithm>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>

#include <unistd.h>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <json.hpp>

#include "../../include/dlx/executor.hpp"
#include "../../include/dlx_program.h"

namespace dlx {

thread_local RunCtx* g_run = nullptr;

void ckc(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Fail(DLX_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void ck(int rc) {
  if (rc != DLX_OK) throw Fail(rc, dlx_last_error());
}

DevVec::~DevVec() {
  if (!wins.empty()) {   // shard windows: freed on their shard's stream (after its readers)
    int cur = 0;
    cudaGetDevice(&cur);
    for (const Win& w : wins) {
      cudaSetDevice(w.dev);
      cudaFreeAsync(w.p, w.st);
    }
    cudaSetDevice(cur);
  }
  if (!p || borrowed) return;
  if (g_run && g_run->fence) (*g_run->fence)();   // a loop still in flight may read this buffer
  cudaFreeAsync(p, fst);
}

// ---- per-thread, per-device resources (kept across runs) -----------------------------------
void* PinnedArena::get(size_t bytes) {
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
void PinnedArena::reset() {   // nothing in flight: keep one block, as large as the run needed
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

DeviceRes& device_res(int device) {
  thread_local std::map<int, DeviceRes> res;   // never torn down (process-lifetime streams)
  DeviceRes& r = res[device];
  if (!r.init) {
    ckc(cudaStreamCreateWithFlags(&r.main, cudaStreamNonBlocking), "cudaStreamCreate");
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

std::string format_val(const Val& x) {
  if (x.is_int()) return std::to_string(x.i());
  if (x.is_dbl()) return format_double(x.d());
  if (x.is_bool()) return x.b() ? "true" : "false";
  if (auto s = std::get_if<std::string>(&x.v)) return *s;
  if (x.is_vec()) return "<vector of " + std::to_string(x.vec()->n) + ">";
  return "()";
}

// ---- executor: construction, pending loops, lazies -------------------------------------------
static std::shared_ptr<Scratch> take_scratch(const Program& p) {
  {
    std::lock_guard<std::mutex> lk(p.scratch_mu);
    if (!p.scratch.empty()) {
      auto s = std::static_pointer_cast<Scratch>(p.scratch.back());
      p.scratch.pop_back();
      return s;
    }
  }
  auto s = std::make_shared<Scratch>();
  s->env.resize(p.max_sym + 1);
  s->bound.assign(p.max_sym + 1, 0);
  s->skip.assign(p.max_sym + 1, 0);
  return s;
}

Executor::Executor(const Program& p, const ExecOpts& o, cudaStream_t st, DeviceRes* res)
    : P(p), opts_(o), st_(st), res_(res), lst_(st), sc_(take_scratch(p)), env_(sc_->env), bound_(sc_->bound),
      skip_(sc_->skip) {
  fence_ = [this] { fence(); };
  if (o.ndevices >= 1 && o.devices)
    devs_.assign(o.devices, o.devices + o.ndevices);
  else
    devs_.push_back(0);
  primary_ = devs_[0];
  replicate_ = getenv("DLX_SHARD_REPLICATE") != nullptr && atoi(getenv("DLX_SHARD_REPLICATE")) != 0;
}

Executor::~Executor() {
  try {
    join_all();
  } catch (...) {
  }
  for (int s : sc_->touched) {   // release this run's values (device vectors are freed here)
    env_[s] = Val{};
    bound_[s] = 0;
    skip_[s] = 0;
  }
  sc_->touched.clear();
  if (!xevents_.empty()) {
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto [dev, e] : xevents_) {
      cudaSetDevice(dev);
      cudaEventSynchronize(e);
      cudaEventDestroy(e);
    }
    cudaSetDevice(cur);
  }
  std::lock_guard<std::mutex> lk(P.scratch_mu);
  if (P.scratch.size() < 2) P.scratch.push_back(sc_);
}

Val Executor::run() {
  if (g_run->profile && !g_run->dry) {
    cudaEventCreate(&prof_t0_);
    cudaEventRecord(prof_t0_, st_);
  }
  Val v = exec_block(P.root);
  join_all();
  return v;
}

std::string Executor::output() const {
  std::string out;
  for (const std::string& l : lines_) {
    out += l;
    out += '\n';
  }
  return out;
}

cudaEvent_t Executor::get_event() {
  if (res_->events.empty()) {
    cudaEvent_t e;
    ckc(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    return e;
  }
  cudaEvent_t e = res_->events.back();
  res_->events.pop_back();
  return e;
}

// The loop just enqueued on lst_ completes at the returned event.  Deferred-binding loops
// (generic kernel: traps, appended lengths) keep `outs` unbound until then, so the first
// statement that reads one of them joins; eager families bind lazies / device vectors at launch.
cudaEvent_t Executor::complete_loop(const std::vector<int>& deferred_outs, std::function<void()> fn) {
  for (int o : deferred_outs) bound_[o] = 0;
  cudaEvent_t ev = get_event();
  ckc(cudaEventRecord(ev, lst_), "cudaEventRecord");
  pending_.push_back(Pending{ev, std::move(fn)});
  return ev;
}

// Device-side ordering only: later main-stream work (frees, host->device rewrites of vectors a
// pending loop may read: the DEG's anti-dependences) waits for every loop in flight.
void Executor::fence() {
  for (const Pending& p : pending_) cudaStreamWaitEvent(st_, p.ev, 0);
}
void Executor::fence_on(cudaStream_t s) {
  for (const Pending& p : pending_) cudaStreamWaitEvent(s, p.ev, 0);
}

void Executor::join_all() {
  if (pending_.empty() && unresolved_.empty() && !main_async_) return;
  const auto t0 = std::chrono::steady_clock::now();
  struct Prof {
    std::chrono::steady_clock::time_point t0;
    size_t n;
    ~Prof() {
      if (g_run && g_run->profile)
        fprintf(stderr, "[dlx profile] @%.2f ms join of %zu loops %.1f us\n", g_run->ms(), n,
                std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
    }
  } prof{t0, pending_.size()};
  std::vector<Pending> pend;
  pend.swap(pending_);
  cudaError_t err = cudaSuccess;
  for (const Pending& p : pend) {
    cudaError_t e = cudaEventSynchronize(p.ev);
    if (err == cudaSuccess) err = e;
    res_->events.push_back(p.ev);
  }
  cudaError_t e = cudaStreamSynchronize(st_);   // main-stream element reads / staged uploads
  if (err == cudaSuccess) err = e;
  main_async_ = false;
  struct ArenaReset {   // the staged results are consumed below (or abandoned on a trap)
    PinnedArena& a;
    ~ArenaReset() { a.reset(); }
  } arena_reset{res_->pin};
  ckc(err, "loop completion");
  for (Pending& p : pend)
    if (p.finish) p.finish();   // program order: the first loop's trap wins
  for (const LazyP& l : unresolved_) {
    if (l->ready) continue;
    int64_t b = 0;
    if (l->esz == 8) std::memcpy(&b, l->src, 8);
    else if (l->esz == 4) { int32_t w; std::memcpy(&w, l->src, 4); b = w; }
    else b = *l->src;
    l->bits = b;
    l->ready = true;
    l->src = nullptr;
  }
  unresolved_.clear();
  format_prints();
  prints_.clear();
  size_t live = 0;
  for (auto& w : vecs_)
    if (auto v = w.lock()) {
      v->wev = nullptr;   // every device write is complete
      v->snap = nullptr;  // (the pinned staging is reset below)
      v->snap_of = nullptr;
      vecs_[live++] = w;
    }
  vecs_.resize(live);
}

// A small persistent pool for host-side work that is embarrassingly parallel: the formatting
// of a loop's printed results (a GDA fit prints d^2 + 2d + 1 values, the C4 program k d
// centroids; std::to_chars is ~80 ns a value, which made the join of such a program the
// largest host cost of its run).
namespace {
class HostPool {
 public:
  static HostPool& get() {
    // never destroyed: its workers stay blocked on the condition variable until the process
    // ends, and destroying a condition variable with waiters blocks (exit would hang)
    static HostPool* p = new HostPool;
    return *p;
  }
  // fn(i) for i in [0, n), in chunks, on the pool's workers and the calling thread
  void parallel_for(size_t n, const std::function<void(size_t, size_t)>& fn) {
    // a forked child inherits the pool object but not its threads: run serially there
    const size_t parts = getpid() == pid_ ? std::min<size_t>(workers_.size() + 1, (n + 255) / 256) : 1;
    if (parts <= 1) {
      fn(0, n);
      return;
    }
    std::unique_lock<std::mutex> call(call_mu_);   // one parallel_for at a time
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      n_ = n;
      parts_ = parts;
      next_ = 1;
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    fn(0, n / parts);   // part 0 on the caller
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return done_ == parts_ - 1; });
    fn_ = nullptr;
  }

 private:
  HostPool() : pid_(getpid()) {
    const unsigned hw = std::thread::hardware_concurrency();
    const unsigned nw = std::min(7u, hw > 1 ? hw - 1 : 0u);
    for (unsigned w = 0; w < nw; ++w) workers_.emplace_back([this] { loop(); });
    for (auto& t : workers_) t.detach();
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return gen_ != seen && fn_ != nullptr && next_ < parts_; });
      seen = gen_;
      while (fn_ != nullptr && next_ < parts_) {
        const size_t part = next_++;
        const auto* fn = fn_;
        const size_t lo = n_ * part / parts_, hi = n_ * (part + 1) / parts_;
        lk.unlock();
        (*fn)(lo, hi);
        lk.lock();
        if (++done_ == parts_ - 1) done_cv_.notify_one();
      }
    }
  }
  pid_t pid_;
  std::vector<std::thread> workers_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(size_t, size_t)>* fn_ = nullptr;
  size_t n_ = 0, parts_ = 0, next_ = 0, done_ = 0;
  uint64_t gen_ = 0;
};
}  // namespace

void Executor::format_prints() {
  static const bool serial = [] {
    const char* e = getenv("DLX_HOST_POOL");
    return e && e[0] == '0';
  }();
  if (serial) {
    for (auto& [line, l] : prints_) lines_[line] = format_val(lazy_val(*l));
    return;
  }
  HostPool::get().parallel_for(prints_.size(), [&](size_t lo, size_t hi) {
    for (size_t q = lo; q < hi; ++q) lines_[prints_[q].first] = format_val(lazy_val(*prints_[q].second));
  });
}

Val Executor::lazy_val(const Lazy& l) {
  switch (l.ty) {
    case Ty::Double: {
      double d;
      std::memcpy(&d, &l.bits, 8);
      return Val{d};
    }
    case Ty::Bool: return Val{l.bits != 0};
    default: return Val{l.bits};
  }
}

LazyP Executor::make_lazy(const void* src, Ty ty, int esz) {
  // a GDA scatter binds d^2 of these per launch: a deque slot each, no allocation or refcount
  Lazy* l = &lazies_.emplace_back();
  l->src = static_cast<const unsigned char*>(src);
  l->ty = ty;
  l->esz = esz;
  unresolved_.push_back(l);
  return l;
}

Val Executor::force(Val v) {
  if (auto lp = std::get_if<LazyP>(&v.v)) {
    if (!(*lp)->ready) join_all();
    return lazy_val(**lp);
  }
  return v;
}

Val Executor::atomv(const Atom& a) {
  switch (a.k) {
    case Atom::Sym: {
      if (a.sym < 0 || a.sym > P.max_sym) gen_fail("x" + std::to_string(a.sym) + " is not a program symbol");
      if (!bound_[a.sym] && !pending_.empty()) join_all();
      if (!bound_[a.sym]) gen_fail("x" + std::to_string(a.sym) + " referenced before definition");
      return env_[a.sym];
    }
    case Atom::Int: return Val{a.i};
    case Atom::Double: return Val{a.d};
    case Atom::Bool: return Val{a.b};
    case Atom::Str: return Val{a.s};
    default: return Val{};
  }
}

VecP Executor::new_vec(int64_t n, Ty elem, cudaStream_t st, bool zero, bool i32) {
  auto v = std::make_shared<DevVec>();
  v->n = n;
  v->elem = elem;
  v->i32 = i32;
  vecs_.push_back(v);
  if (g_run->dry) return v;
  v->fst = st_;
  ckc(cudaMallocAsync(&v->p, std::max<size_t>(16, static_cast<size_t>(n) * v->esize()), st), "cudaMallocAsync");
  if (zero) ckc(cudaMemsetAsync(v->p, 0, static_cast<size_t>(n) * v->esize(), st), "cudaMemset");
  return v;
}

// An Int vector kept as int32 on the device (k-means assignments) becomes int64 before a
// consumer that needs the reference layout (a loop, a host write), on stream s.
void Executor::widen(const VecP& v, cudaStream_t s) {
  if (!v->i32 || g_run->dry) return;
  if (v->wev) cudaStreamWaitEvent(s, v->wev, 0);
  void* w = nullptr;
  ckc(cudaMallocAsync(&w, std::max<int64_t>(2, v->n) * 8, s), "cudaMallocAsync");
  ck(dlx_widen_i32_i64(static_cast<const int32_t*>(v->p), v->n, static_cast<int64_t*>(w), s));
  cudaFreeAsync(v->p, s);
  v->p = w;
  v->i32 = false;
  v->touched();   // same values, new layout: shard windows are stale
  if (s != st_) {   // a loop stream rewrote the buffer: later readers order after it
    cudaEvent_t ev = get_event();
    ckc(cudaEventRecord(ev, s), "cudaEventRecord");
    pending_.push_back(Pending{ev, nullptr});
    v->wev = ev;
  }
}

// ---- host mirrors of small vectors ---------------------------------------------------------
// Small vectors (<= kMirrorBytes: centroids, counts, sums, parameters) keep a host mirror so
// host statements that read or update them element by element (VectorApply / VectorUpdate)
// cost one transfer per vector instead of one synchronous copy per element: the mirror is
// loaded on the first host read, host writes mark a dirty range, and every loop launch first
// flushes dirty ranges (asynchronously, through pinned staging).  Loops invalidate the mirror
// of every vector they write.
void Executor::load_mirror(const VecP& v) {
  if (v->host_valid) return;
  if (v->wev) join_all();
  const size_t hs = v->hsize();
  v->host.resize(static_cast<size_t>(v->n) * hs);
  if (!v->host.empty()) {
    if (v->i32) {
      std::vector<int32_t> tmp(v->n);
      ckc(cudaMemcpyAsync(tmp.data(), v->p, v->n * 4, cudaMemcpyDeviceToHost, st_), "d2h");
      ckc(cudaStreamSynchronize(st_), "sync");
      for (int64_t i = 0; i < v->n; ++i) {
        const int64_t w = tmp[i];
        std::memcpy(v->host.data() + i * 8, &w, 8);
      }
    } else {
      ckc(cudaMemcpyAsync(v->host.data(), v->p, v->host.size(), cudaMemcpyDeviceToHost, st_), "d2h");
      ckc(cudaStreamSynchronize(st_), "sync");
    }
  }
  v->host_valid = true;
}

void Executor::flush_mirrors() {   // before a loop launch: host updates -> device
  bool any = false;
  for (auto& w : vecs_)
    if (auto v = w.lock())
      if (v->dirty_hi > v->dirty_lo) {
        if (!any) fence();   // WAR: a loop in flight may still read the old contents
        any = true;
        const size_t es = v->esize();
        const size_t bytes = static_cast<size_t>(v->dirty_hi - v->dirty_lo) * es;
        void* stage = res_->pin.get(bytes);
        std::memcpy(stage, v->host.data() + v->dirty_lo * es, bytes);
        ckc(cudaMemcpyAsync(static_cast<unsigned char*>(v->p) + v->dirty_lo * es, stage, bytes,
                            cudaMemcpyHostToDevice, st_), "h2d");
        main_async_ = true;
        v->dirty_lo = INT64_MAX;
        v->dirty_hi = -1;
      }
}

Val Executor::host_elem(const unsigned char* h, Ty elem) {
  if (elem == Ty::Double) {
    double x;
    std::memcpy(&x, h, 8);
    return Val{x};
  }
  if (elem == Ty::Bool) return Val{*h != 0};
  int64_t x;
  std::memcpy(&x, h, 8);
  return Val{x};
}

Val Executor::vec_get(const VecP& v, int64_t i) {
  if (i < 0 || i >= v->n) trap("TrapIndexOutOfBounds: index " + std::to_string(i));
  if (g_run->dry) return v->elem == Ty::Double ? Val{0.5} : v->elem == Ty::Bool ? Val{false} : Val{int64_t{1}};
  if (v->wev) join_all();
  if (v->mirrored()) {
    load_mirror(v);
    return host_elem(v->host.data() + static_cast<size_t>(i) * v->hsize(), v->elem);
  }
  // large vectors: a read-through page of host copies around the element (host statements
  // that read x(0), x(1), ... — the k-means centroid initialisation — cost one transfer per
  // page instead of one synchronous copy per element)
  const size_t es = v->esize();
  if (!v->page_valid || i < v->page_lo || i >= v->page_lo + static_cast<int64_t>(v->page.size() / es)) {
    const int64_t lo = i & ~(kPageElems - 1), hi = std::min(v->n, lo + kPageElems);
    v->page.resize(static_cast<size_t>(hi - lo) * es);
    ckc(cudaMemcpyAsync(v->page.data(), static_cast<unsigned char*>(v->p) + lo * es, v->page.size(),
                        cudaMemcpyDeviceToHost, st_), "d2h");
    ckc(cudaStreamSynchronize(st_), "sync");
    v->page_lo = lo;
    v->page_valid = true;
  }
  const unsigned char* h = v->page.data() + static_cast<size_t>(i - v->page_lo) * es;
  if (v->i32) {
    int32_t w;
    std::memcpy(&w, h, 4);
    return Val{static_cast<int64_t>(w)};
  }
  return host_elem(h, v->elem);
}

void Executor::vec_set(const VecP& v, int64_t i, const Val& x) {
  if (i < 0 || i >= v->n) trap("TrapIndexOutOfBounds: store index " + std::to_string(i));
  if (g_run->dry) return;
  v->touched();
  if (v->i32) {   // the host writes reference Ints: widen the device copy first
    fence();
    widen(v, st_);
    v->host_valid = false;
    v->page_valid = false;
  }
  auto encode = [&](unsigned char* h) {
    if (v->elem == Ty::Double) {
      const double d = x.d();
      std::memcpy(h, &d, 8);
    } else if (v->elem == Ty::Bool) {
      *h = x.b() ? 1 : 0;
    } else {
      const int64_t q = x.i();
      std::memcpy(h, &q, 8);
    }
  };
  if (v->mirrored()) {
    load_mirror(v);
    encode(v->host.data() + static_cast<size_t>(i) * v->hsize());
    v->dirty_lo = std::min(v->dirty_lo, i);
    v->dirty_hi = std::max(v->dirty_hi, i + 1);
    return;
  }
  if (v->wev) join_all();
  fence();
  v->page_valid = false;   // the page may hold the old value
  auto* stage = static_cast<unsigned char*>(res_->pin.get(8));
  encode(stage);
  ckc(cudaMemcpyAsync(static_cast<unsigned char*>(v->p) + i * v->esize(), stage, v->esize(), cudaMemcpyHostToDevice, st_),
      "h2d");
  main_async_ = true;
}

// ---- host interpretation ---------------------------------------------------------------------
Val Executor::exec_block(int b) {
  const Block& bl = P.block(b);
  for (int s : bl.stmts) {
    if (skip_[s]) {   // executed on the device by the preceding loop's launch (UpdateGroup)
      skip_[s] = 0;
      continue;
    }
    const Stmt& st = P.stmts[s];
    try {
      if (!g_run->dry && !P.copy_runs.empty()) {
        auto cr = P.copy_runs.find(s);
        if (cr != P.copy_runs.end() && copy_run(cr->second)) continue;   // the run is now skipped
      }
      if (st.op == Op::ParallelLoop) {
        run_loop(st);   // binds every live elem's `out` (elems[0].out is the statement's own sym)
      } else {
        bind(s, exec_stmt(st));
      }
    } catch (...) {
      join_all();   // a trap of an earlier loop still in flight takes precedence
      throw;
    }
  }
  return atomv(bl.result);
}

// A CopyRun as device copies on the main stream (ordered after its producers and before the
// next loop launch like any host write); false -> run its statements on the host (a trap, a
// type mismatch, int32 storage: the host path reports exactly what the reference would).
bool Executor::copy_run(const CopyRun& run) {
  if (!bound_[run.x_sym] || !bound_[run.v_sym]) return false;
  const Val& xv = env_[run.x_sym];
  const Val& vv = env_[run.v_sym];
  if (!xv.is_vec() || !vv.is_vec()) return false;
  const VecP& X = xv.vec();
  const VecP& V = vv.vec();
  if (X == V || X->elem != V->elem || X->i32 || V->i32) return false;
  for (auto [e1, e2] : run.pairs)
    if (e1 < 0 || e1 >= X->n || e2 < 0 || e2 >= V->n) return false;
  flush_mirrors();   // V's earlier host writes land first
  fence();           // WAR: loops in flight may read V
  if (X->wev) cudaStreamWaitEvent(st_, X->wev, 0);
  if (V->wev) cudaStreamWaitEvent(st_, V->wev, 0);
  const size_t es = X->esize();
  size_t q = 0;
  while (q < run.pairs.size()) {   // coalesce runs of consecutive (e1, e2)
    size_t r = q + 1;
    while (r < run.pairs.size() && run.pairs[r].first == run.pairs[r - 1].first + 1 &&
           run.pairs[r].second == run.pairs[r - 1].second + 1)
      ++r;
    ckc(cudaMemcpyAsync(static_cast<unsigned char*>(V->p) + run.pairs[q].second * es,
                        static_cast<const unsigned char*>(X->p) + run.pairs[q].first * es, (r - q) * es,
                        cudaMemcpyDeviceToDevice, st_), "d2d copy run");
    q = r;
  }
  V->host_valid = false;
  V->page_valid = false;
  V->touched();
  for (size_t t = 1; t < run.stmts.size(); ++t) mark_skip(run.stmts[t]);
  return true;
}

static int64_t wrap(uint64_t v) { return static_cast<int64_t>(v); }

Val Executor::scalar(Op op, const Val& x, const Val& y) {
  if (op == Op::And) return Val{x.b() && y.b()};
  if (op == Op::Or) return Val{x.b() || y.b()};
  if (x.is_int() && y.is_int()) {
    const int64_t a = x.i(), b = y.i();
    switch (op) {
      case Op::Plus: return Val{wrap(static_cast<uint64_t>(a) + static_cast<uint64_t>(b))};
      case Op::Minus: return Val{wrap(static_cast<uint64_t>(a) - static_cast<uint64_t>(b))};
      case Op::Times: return Val{wrap(static_cast<uint64_t>(a) * static_cast<uint64_t>(b))};
      case Op::Divide:
        if (b == 0) trap("TrapDivByZero: integer division by zero");
        return Val{(a == INT64_MIN && b == -1) ? a : a / b};
      case Op::Lt: return Val{a < b};
      case Op::Eq: return Val{a == b};
      default: break;
    }
  }
  if (x.is_dbl() && y.is_dbl()) {
    const double a = x.d(), b = y.d();
    switch (op) {
      case Op::Plus: return Val{a + b};
      case Op::Minus: return Val{a - b};
      case Op::Times: return Val{a * b};
      case Op::Divide: return Val{a / b};
      case Op::Lt: return Val{a < b};
      case Op::Eq: return Val{a == b};
      default: break;
    }
  }
  if (op == Op::Eq) return Val{x.v == y.v};
  gen_fail("don't know how to evaluate this operator on these operand types");
}

Val Executor::exec_stmt(const Stmt& s) {
  switch (s.op) {
    case Op::Plus: case Op::Minus: case Op::Times: case Op::Divide: case Op::Lt: case Op::Eq:
    case Op::And: case Op::Or:
      return scalar(s.op, atom(s.args[0]), atom(s.args[1]));
    case Op::Not: return Val{!atom(s.args[0]).b()};
    case Op::MathAbs: {
      Val x = atom(s.args[0]);
      if (x.is_int()) return Val{x.i() < 0 ? wrap(0ull - static_cast<uint64_t>(x.i())) : x.i()};
      return Val{std::fabs(x.d())};
    }
    case Op::MathSqrt: return Val{std::sqrt(atom(s.args[0]).d())};
    case Op::MathExp: return Val{std::exp(atom(s.args[0]).d())};
    case Op::ToDouble: return Val{static_cast<double>(atom(s.args[0]).i())};
    case Op::IfThenElse: return exec_block(atom(s.args[0]).b() ? s.blocks[0] : s.blocks[1]);
    case Op::While:
      while (force(exec_block(s.blocks[0])).b()) exec_block(s.blocks[1]);
      return Val{};
    case Op::VarAlloc: {
      auto c = std::make_shared<Cell>();
      c->v = atomv(s.args[0]);
      return Val{c};
    }
    case Op::VarRead: return std::get<CellP>(atomv(s.args[0]).v)->v;
    case Op::VarWrite:
      std::get<CellP>(atomv(s.args[0]).v)->v = atomv(s.args[1]);
      return Val{};
    case Op::Print: {
      Val x = atomv(s.args[0]);
      if (auto lp = std::get_if<LazyP>(&x.v); lp && !(*lp)->ready) {
        prints_.emplace_back(lines_.size(), *lp);   // filled in when the loop's result arrives
        lines_.emplace_back();
      } else {
        lines_.push_back(format_val(force(x)));
      }
      return Val{};
    }
    case Op::VectorRand: case Op::VectorRandInt: {
      const int64_t n = atom(s.args[0]).i();
      const bool ints = s.op == Op::VectorRandInt;
      const Ty et = ints ? Ty::Int : Ty::Double;
      if (n < 0) trap("TrapIndexOutOfBounds: negative vector length");
      const dlx_program_input* in = nullptr;
      for (int q = 0; q < opts_.ninputs; ++q)
        if (opts_.inputs[q].sym == s.sym) in = &opts_.inputs[q];
      VecP v;
      if (in) {   // caller-supplied data for this source (the draw counter still advances)
        if (in->n != n || in->elem != (ints ? DLX_VAL_INT : DLX_VAL_DOUBLE) || (!in->h_data && !in->d_data))
          throw Fail(DLX_ERR_ARG, "input for x" + std::to_string(s.sym) + " does not match the statement (length " +
                                      std::to_string(n) + ", " + (ints ? "Int" : "Double") + ")");
        if (in->d_data) {
          v = std::make_shared<DevVec>();
          v->n = n;
          v->elem = et;
          v->p = in->d_data;
          v->borrowed = true;
          vecs_.push_back(v);
        } else {
          v = new_vec(n, et, st_, false);
          if (!g_run->dry && n > 0) {
            ckc(cudaMemcpyAsync(v->p, in->h_data, static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice, st_), "h2d input");
            main_async_ = true;
          }
        }
      } else {
        v = new_vec(n, et, st_, false);
        v->gen = true;
        v->gen_int = ints;
        v->gen_seed = opts_.seed;
        v->gen_first = draws_;
        v->gen_bound = ints ? atom(s.args[1]).i() : 0;
        if (g_run->dry) {
        } else if (ints) {
          ck(dlx_rng_ints(static_cast<int64_t*>(v->p), n, atom(s.args[1]).i(), opts_.seed, draws_, st_));
        } else {
          ck(dlx_rng_units(static_cast<double*>(v->p), n, opts_.seed, draws_, st_));
        }
      }
      draws_ += static_cast<uint64_t>(n);
      return Val{v};
    }
    case Op::VectorNew: {
      const Ty e = s.aux_ty.t;
      if (e != Ty::Int && e != Ty::Double && e != Ty::Bool) gen_fail("vectors of Str / records / vectors");
      const int64_t n = atom(s.args[0]).i();
      if (n < 0) trap("TrapIndexOutOfBounds: negative vector length");
      return Val{new_vec(n, e, st_, true)};
    }
    case Op::VectorLiteral: {
      const Ty e = s.aux_ty.t == Ty::Double ? Ty::Double : Ty::Int;
      VecP v = new_vec(static_cast<int64_t>(s.lits.size()), e, st_, false);
      if (!g_run->dry && !s.lits.empty()) {
        auto* raw = static_cast<int64_t*>(res_->pin.get(s.lits.size() * 8));
        for (size_t q = 0; q < s.lits.size(); ++q) {
          if (e == Ty::Double) {
            const double d = s.lits[q].k == Atom::Double ? s.lits[q].d : static_cast<double>(s.lits[q].i);
            std::memcpy(&raw[q], &d, 8);
          } else {
            raw[q] = s.lits[q].i;
          }
        }
        ckc(cudaMemcpyAsync(v->p, raw, s.lits.size() * 8, cudaMemcpyHostToDevice, st_), "h2d");
        main_async_ = true;
      }
      return Val{v};
    }
    case Op::VectorLength: return Val{vec_of(s.args[0])->n};
    case Op::VectorApply: {
      VecP v = vec_of(s.args[0]);
      const int64_t i = atom(s.args[1]).i();
      if (i < 0 || i >= v->n) trap("TrapIndexOutOfBounds: index " + std::to_string(i));
      if (v->wev && !g_run->dry && P.print_only[s.sym]) {
        // a printed element of a vector a loop is still writing: read it asynchronously (small
        // vectors: one snapshot of the whole vector serves every such read until the next join)
        if (v->mirrored()) {
          if (!v->snap || v->snap_of != v->wev) {
            cudaStreamWaitEvent(st_, v->wev, 0);
            auto* stage = static_cast<unsigned char*>(res_->pin.get(std::max<size_t>(1, v->n * v->esize())));
            ckc(cudaMemcpyAsync(stage, v->p, v->n * v->esize(), cudaMemcpyDeviceToHost, st_), "d2h");
            v->snap = stage;
            v->snap_of = v->wev;
            main_async_ = true;
          }
          return Val{make_lazy(v->snap + i * v->esize(), v->elem, static_cast<int>(v->esize()))};
        }
        cudaStreamWaitEvent(st_, v->wev, 0);
        auto* stage = res_->pin.get(8);
        ckc(cudaMemcpyAsync(stage, static_cast<unsigned char*>(v->p) + i * v->esize(), v->esize(), cudaMemcpyDeviceToHost,
                            st_), "d2h");
        main_async_ = true;
        return Val{make_lazy(stage, v->elem, static_cast<int>(v->esize()))};
      }
      return vec_get(v, i);
    }
    case Op::VectorUpdate:
      vec_set(vec_of(s.args[0]), atom(s.args[1]).i(), atom(s.args[2]));
      return Val{};
    case Op::ParallelLoop: run_loop(s); return Val{};
    default: break;
  }
  gen_fail("don't know how to generate code for: " + s.opname + " (x" + std::to_string(s.sym) + ")");
}

VecP Executor::vec_of(const Atom& a) {
  Val v = atomv(a);
  if (!v.is_vec()) gen_fail("expected a vector");
  return v.vec();
}

}  // namespace dlx

// ---- API ------------------------------------------------------------------------------------
namespace dlx {

struct ProgramHandle {
  std::shared_ptr<const Program> prog;
};

namespace {

std::shared_ptr<const Program> cached_program(const char* text, size_t len) {
  // parsed descriptors by content for dlx_program_run (a caller that runs the same staged
  // program again skips the parse); handles (dlx_program_create) are the cheaper way
  static std::mutex mu;
  static std::unordered_map<std::string, std::shared_ptr<const Program>> cache;
  static std::vector<std::string> order;
  std::string key(text, len);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  std::shared_ptr<const Program> p = parse_program(text, len);
  std::lock_guard<std::mutex> lk(mu);
  if (cache.emplace(key, p).second) {
    order.push_back(key);
    if (order.size() > 8) {
      cache.erase(order.front());
      order.erase(order.begin());
    }
  }
  return p;
}

struct RunOut {
  std::string text, report;
  Val result;
  // vector results downloaded to the host
  int32_t vec_elem = 0;
  std::vector<unsigned char> vec;
  int64_t vec_len = 0;
};

RunOut execute(const Program& p, const ExecOpts& o) {
  RunCtx ctx;
  ctx.dry = (o.flags & DLX_EXEC_DRYRUN) || getenv("DLX_PROGRAM_DRYRUN") != nullptr;
  ctx.debug = getenv("DLX_PROGRAM_DEBUG") != nullptr;
  ctx.serial = (o.flags & DLX_EXEC_SERIAL) || getenv("DLX_PROGRAM_SERIAL") != nullptr;
  ctx.nocache = (o.flags & DLX_EXEC_NOCACHE) != 0;
  ctx.profile = getenv("DLX_PROGRAM_PROFILE") != nullptr;
  ctx.t0 = std::chrono::steady_clock::now();
  const auto t_run = std::chrono::steady_clock::now();
  const int device = (o.ndevices >= 1 && o.devices) ? o.devices[0] : 0;
  if (o.ndevices > 1 && !ctx.dry) {   // sharded loops (shard.cpp): every device must exist
    int count = 0;
    ckc(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    for (int g = 0; g < o.ndevices; ++g)
      if (o.devices[g] < 0 || o.devices[g] >= count)
        throw Fail(DLX_ERR_ARG, "ExecOptions.devices[" + std::to_string(g) + "] = " + std::to_string(o.devices[g]) +
                                    " is not a device (" + std::to_string(count) + " visible)");
    for (int g = 1; g < o.ndevices; ++g)   // peer access where the hardware offers it (NVLink)
      if (o.devices[g] != device) {
        int can = 0;
        cudaDeviceCanAccessPeer(&can, device, o.devices[g]);
        if (can) {
          cudaSetDevice(device);
          cudaDeviceEnablePeerAccess(o.devices[g], 0);
          cudaSetDevice(o.devices[g]);
          cudaDeviceEnablePeerAccess(device, 0);
          cudaGetLastError();   // already enabled: not an error here
        }
      }
  }
  DeviceRes* res = nullptr;
  cudaStream_t st = nullptr;
  if (!ctx.dry) {
    ckc(cudaSetDevice(device), "cudaSetDevice");
    res = &device_res(device);
    st = res->main;
  }
  ctx.main = st;
  struct CtxGuard {
    RunCtx* prev;
    explicit CtxGuard(RunCtx* c) : prev(g_run) { g_run = c; }
    ~CtxGuard() { g_run = prev; }
  } guard(&ctx);
  RunOut out;
  {
    DeviceRes dry_res;
    Executor ex(p, o, st, ctx.dry ? &dry_res : res);
    ctx.fence = ctx.dry ? nullptr : &ex.fence_;
    Val v = ex.run();
    if (ctx.profile) fprintf(stderr, "[dlx profile] @%.2f ms program done\n", ctx.ms());
    out.text = ex.output();
    out.report = ex.report.dump();
    v = ex.force(v);
    if (v.is_vec() && !ctx.dry) {   // RunResult.result holds the vector (runtime.hpp:100-103)
      const VecP& vec = v.vec();
      out.vec_len = vec->n;
      out.vec_elem = vec->elem == Ty::Double ? DLX_VAL_DOUBLE : vec->elem == Ty::Bool ? DLX_VAL_BOOL : DLX_VAL_INT;
      out.vec.resize(static_cast<size_t>(vec->n) * vec->hsize());
      if (vec->n > 0) {
        if (vec->i32) ex.widen(vec, st);
        ckc(cudaMemcpyAsync(out.vec.data(), vec->p, out.vec.size(), cudaMemcpyDeviceToHost, st), "d2h result");
        ckc(cudaStreamSynchronize(st), "sync");
      }
    }
    out.result = v;
    ex.join_all();
    if (ctx.profile) fprintf(stderr, "[dlx profile] @%.2f ms results out\n", ctx.ms());
  }
  if (ctx.profile) fprintf(stderr, "[dlx profile] @%.2f ms executor released\n", ctx.ms());
  if (!ctx.dry) ckc(cudaStreamSynchronize(st), "sync");
  if (ctx.profile)
    fprintf(stderr, "[dlx profile] run %.1f us\n",
            std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_run).count());
  return out;
}

int fail_code(const Fail& f) { return f.code; }

}  // namespace

RunResult run_program(const std::string& program_json, uint64_t seed, int device) {
  std::shared_ptr<const Program> p;
  try {
    p = cached_program(program_json.data(), program_json.size());
    ExecOpts o{};
    o.seed = seed;
    o.ndevices = 1;
    o.devices = &device;
    RunOut r = execute(*p, o);
    RunResult rr;
    rr.output = std::move(r.text);
    rr.result = format_val(r.result);
    rr.report = std::move(r.report);
    return rr;
  } catch (const Fail& f) {
    if (f.code == DLX_ERR_GENERATION) throw GenerationFailed(f.what());
    if (f.code == DLX_ERR_TRAP) throw TrapError(f.what());
    throw std::runtime_error(f.what());
  }
}

}  // namespace dlx

using namespace dlx;

extern "C" {

int dlx_program_create(const char* program_json, size_t len, dlx_program_t* out) {
  if (!program_json || !out) {
    set_error("dlx_program_create: null argument");
    return DLX_ERR_ARG;
  }
  try {
    auto* h = new ProgramHandle{parse_program(program_json, len ? len : strlen(program_json))};
    *out = reinterpret_cast<dlx_program_t>(h);
    return DLX_OK;
  } catch (const Fail& f) {
    set_error("%s", f.what());
    return fail_code(f);
  } catch (const std::exception& e) {
    set_error("dlx_program_create: malformed descriptor: %s", e.what());
    return DLX_ERR_ARG;
  }
}

int dlx_program_destroy(dlx_program_t program) {
  delete reinterpret_cast<ProgramHandle*>(program);
  return DLX_OK;
}

static char* dup_str(const std::string& s) {
  char* r = static_cast<char*>(malloc(s.size() + 1));
  if (r) std::memcpy(r, s.c_str(), s.size() + 1);
  return r;
}

int dlx_program_execute(dlx_program_t program, const dlx_exec_options* opts, dlx_run_result* out) {
  if (!program || !out) {
    set_error("dlx_program_execute: null argument");
    return DLX_ERR_ARG;
  }
  std::memset(out, 0, sizeof(*out));
  ExecOpts o{};
  o.seed = 1;
  if (opts) o = *opts;
  try {
    RunOut r = execute(*reinterpret_cast<ProgramHandle*>(program)->prog, o);
    out->text = dup_str(r.text);
    out->report = dup_str(r.report);
    out->s = dup_str(format_val(r.result));
    const Val& v = r.result;
    if (v.is_int()) out->kind = DLX_VAL_INT, out->i = v.i();
    else if (v.is_dbl()) out->kind = DLX_VAL_DOUBLE, out->d = v.d();
    else if (v.is_bool()) out->kind = DLX_VAL_BOOL, out->i = v.b();
    else if (std::holds_alternative<std::string>(v.v)) out->kind = DLX_VAL_STR;
    else if (v.is_vec()) {
      out->kind = DLX_VAL_VECTOR;
      out->vec_elem = r.vec_elem;
      out->vec_len = r.vec_len;
      out->vec_data = malloc(std::max<size_t>(1, r.vec.size()));
      if (!r.vec.empty()) std::memcpy(out->vec_data, r.vec.data(), r.vec.size());
    } else {
      out->kind = DLX_VAL_UNIT;
    }
    return DLX_OK;
  } catch (const Fail& f) {
    set_error("%s", f.what());
    return fail_code(f);
  } catch (const nlohmann::json::exception& e) {
    set_error("dlx_program_execute: malformed descriptor: %s", e.what());
    return DLX_ERR_ARG;
  } catch (const std::exception& e) {
    set_error("%s", e.what());
    return DLX_ERR_CUDA;
  }
}

void dlx_run_result_free(dlx_run_result* r) {
  if (!r) return;
  free(r->text);
  free(r->report);
  free(r->s);
  free(r->vec_data);
  std::memset(r, 0, sizeof(*r));
}

int dlx_program_run(const char* program_json, uint64_t seed, int device, char** out_text, char** out_report) {
  if (!program_json || !out_text) {
    set_error("dlx_program_run: null argument");
    return DLX_ERR_ARG;
  }
  try {
    std::shared_ptr<const Program> p = cached_program(program_json, strlen(program_json));
    ExecOpts o{};
    o.seed = seed;
    o.ndevices = 1;
    o.devices = &device;
    RunOut r = execute(*p, o);
    *out_text = dup_str(r.text);
    if (out_report) *out_report = dup_str(r.report);
    return DLX_OK;
  } catch (const Fail& f) {
    set_error("%s", f.what());
    return fail_code(f);
  } catch (const nlohmann::json::exception& e) {
    set_error("dlx_program_run: malformed descriptor: %s", e.what());
    return DLX_ERR_ARG;
  } catch (const std::exception& e) {
    set_error("%s", e.what());
    return DLX_ERR_CUDA;
  }
}

void dlx_string_free(char* s) { free(s); }

}  // extern "C"
