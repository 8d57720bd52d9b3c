// shard.cpp — multi-device execution of the drop-in (ExecOptions.devices):
// the lift of executeDEG's workers and contiguous chunks to devices.  One host
// thread drives every device (SPEC.md: one controlling thread per DEG instance).  A root loop of
// a sharded family runs as G contiguous index shards (boundaries n g / G rounded down to 64), shard g on
// devices[g]; each shard's partial record (counts, sums, gradient, scatter) is folded into the
// primary device's (devices[0]) in ascending shard order — the executor's ascending-chunk
// combine, so results do not depend on which device finished first — and
// collect outputs (assignments, h) land in the primary's vector at the shard's offset.
//
// Inputs reach a shard's device as windows: the element range the shard reads (rows
// [lo, hi) of x, the whole centroid / theta vector), cached per vector and shard until the
// vector is written.  A window of a synthetic source (VectorRand / VectorRandInt never written
// since) is drawn on the shard's device by LCG skip-ahead — bit-identical, and no primary copy
// crosses NVLink; any other window is a peer copy from the primary.  On the primary itself a
// window is the vector (no copy) unless DLX_SHARD_REPLICATE=1 (tests: the window path on one GPU).
//
// Families: kmeans (fold fused with the centroid update), groupby, bucket_rows (GDA pass 1),
// gda_scatter (GDA pass 2), logistic (fold, then the theta update).  Compiled generic loops run
// on the primary device (their index expressions are not known to be row-affine).
#include <cstring>

#include "program_exec.hpp"

namespace dlx {

// fold kernels (combine.cu): partial records in ascending order
int combine_f64(const double* parts, int nparts, long long width, double* out, cudaStream_t s);
int combine_f64_i64(const double* pf, long long wf, double* of, const long long* pi, long long wi,
                    long long* oi, int nparts, cudaStream_t s);
int combine_kmeans_update(const double* pf, double* of, const long long* pi, long long* oi, int k, int d,
                          int nparts, double* mu, cudaStream_t s);

namespace {
[[noreturn]] void load_trap() { trap("TrapIndexOutOfBounds: element load out of range in a multiloop"); }
}  // namespace

bool Executor::sharded(const LoopPlan& p) const {
  if (devs_.size() <= 1) return false;
  switch (p.fam) {
    case LoopPlan::Kmeans: case LoopPlan::GroupBy: case LoopPlan::BucketRows: case LoopPlan::GdaScatter:
    case LoopPlan::Logistic: return true;
    default: return false;
  }
}

std::vector<Executor::Shard> Executor::shards(int64_t n) {
  const int G = static_cast<int>(devs_.size());
  std::vector<Shard> sh;
  for (int g = 0; g < G; ++g) {
    Shard s;
    s.g = g;
    s.dev = devs_[g];
    // boundaries on multiples of 64 indices: every shard's rows start 512-byte aligned (the
    // kernels' vector loads and bulk copies need 16-byte aligned rows and keys)
    s.lo = g == 0 ? 0 : (n * g / G) & ~int64_t{63};
    s.hi = g == G - 1 ? n : (n * (g + 1) / G) & ~int64_t{63};
    s.local = s.dev == primary_ && !replicate_;
    if (s.dev == primary_) s.st = g == 0 ? lst_ : res_->loop[(launches_ + g) % kLoopStreams];
    else {
      ckc(cudaSetDevice(s.dev), "cudaSetDevice");
      s.st = device_res(s.dev).loop[g % kLoopStreams];
      ckc(cudaSetDevice(primary_), "cudaSetDevice");
    }
    sh.push_back(s);
  }
  return sh;
}

cudaEvent_t Executor::dev_event(int dev) {
  cudaEvent_t e;
  ckc(cudaSetDevice(dev), "cudaSetDevice");
  ckc(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
  xevents_.emplace_back(dev, e);
  return e;
}

// elements [lo, hi) of v on shard s's device (the current device is s.dev)
const void* Executor::window(const VecP& v, const Shard& s, int64_t lo, int64_t hi) {
  const size_t es = v->esize();
  if (s.local) return static_cast<const unsigned char*>(v->p) + lo * es;
  for (const DevVec::Win& w : v->wins)
    if (w.shard == s.g && w.dev == s.dev && w.ver == v->ver && w.lo <= lo && hi <= w.hi)
      return static_cast<const unsigned char*>(w.p) + (lo - w.lo) * es;
  for (auto it = v->wins.begin(); it != v->wins.end();)   // this shard's stale window
    if (it->shard == s.g) {
      cudaFreeAsync(it->p, it->st);
      it = v->wins.erase(it);
    } else {
      ++it;
    }
  DevVec::Win w;
  w.shard = s.g;
  w.dev = s.dev;
  w.lo = lo;
  w.hi = hi;
  w.ver = v->ver;
  w.st = s.st;
  const int64_t len = hi - lo;
  ckc(cudaMallocAsync(&w.p, std::max<size_t>(16, static_cast<size_t>(len) * es), s.st), "cudaMallocAsync");
  if (len > 0) {
    if (v->gen && !v->i32) {   // a synthetic source: draw the window here (skip-ahead)
      if (v->gen_int)
        ck(dlx_rng_ints(static_cast<int64_t*>(w.p), len, v->gen_bound, v->gen_seed, v->gen_first + lo, s.st));
      else
        ck(dlx_rng_units(static_cast<double*>(w.p), len, v->gen_seed, v->gen_first + lo, s.st));
    } else {
      ckc(cudaMemcpyPeerAsync(w.p, s.dev, static_cast<const unsigned char*>(v->p) + lo * es, primary_,
                              static_cast<size_t>(len) * es, s.st), "cudaMemcpyPeerAsync window");
    }
  }
  v->wins.push_back(w);
  return w.p;
}

// A sharded loop's skeleton: inputs ready on the primary (`ready`, recorded on lst_), shard
// launches on their devices' streams, then lst_ waits for every shard.
void Executor::run_shards(std::vector<Shard>& sh, const std::function<void(Shard&)>& body) {
  cudaEvent_t ready = get_event();
  ckc(cudaEventRecord(ready, lst_), "cudaEventRecord");
  pending_.push_back(Pending{ready, nullptr});   // recycled at the next join
  for (Shard& s : sh) {
    if (s.st != lst_) ckc(cudaStreamWaitEvent(s.st, ready, 0), "cudaStreamWaitEvent");
    ckc(cudaSetDevice(s.dev), "cudaSetDevice");
    try {
      body(s);
    } catch (...) {
      cudaSetDevice(primary_);
      throw;
    }
    if (s.st != lst_) {
      cudaEvent_t e = dev_event(s.dev);
      ckc(cudaSetDevice(s.dev), "cudaSetDevice");
      ckc(cudaEventRecord(e, s.st), "cudaEventRecord");
      ckc(cudaSetDevice(primary_), "cudaSetDevice");
      ckc(cudaStreamWaitEvent(lst_, e, 0), "cudaStreamWaitEvent");
    }
    ckc(cudaSetDevice(primary_), "cudaSetDevice");
  }
}

// shard-local output buffer: `dst` itself (a local shard), or a buffer on the shard's device
// peer-copied into `dst` after the shard's kernels (copy_back)
static void* shard_buf(const Executor::Shard& s, void* dst, size_t bytes) {
  if (s.local) return dst;
  void* p = nullptr;
  ckc(cudaMallocAsync(&p, std::max<size_t>(16, bytes), s.st), "cudaMallocAsync");
  return p;
}
static void copy_back(const Executor::Shard& s, void* dst, int primary, void* src, size_t bytes) {
  if (s.local) return;
  if (bytes) ckc(cudaMemcpyPeerAsync(dst, primary, src, s.dev, bytes, s.st), "cudaMemcpyPeerAsync");
  cudaFreeAsync(src, s.st);
}

void Executor::launch_kmeans_sharded(LoopPlan& p, int64_t n, std::vector<VecP>& V, nlohmann::json& rep) {
  const VecP& x = V[p.x];
  const VecP& mu = V[p.mu];
  const int d = static_cast<int>(p.d), k = static_cast<int>(p.k);
  if (n * d > x->n || static_cast<int64_t>(k) * d > mu->n) load_trap();
  wait_inputs(V);
  VecP U;
  if (p.upd_vec >= 0 && bound_[p.upd_vec] && env_[p.upd_vec].is_vec()) {
    U = env_[p.upd_vec].vec();
    if (U->elem != Ty::Double || U->n != static_cast<int64_t>(k) * d || U->i32) U = nullptr;
  }
  if (U) {
    fence_on(lst_);
    if (U->wev) cudaStreamWaitEvent(lst_, U->wev, 0);
  }
  std::vector<Shard> sh = shards(n);
  const int G = static_cast<int>(sh.size());
  VecP assign = new_vec(n, Ty::Int, lst_, false, /*i32=*/true);
  auto* pi = static_cast<int64_t*>(dalloc(static_cast<size_t>(G) * k * 8));
  auto* pf = static_cast<double*>(dalloc(static_cast<size_t>(G) * k * d * 8));
  run_shards(sh, [&](Shard& s) {
    const int64_t ng = s.hi - s.lo;
    int64_t* cd = pi + static_cast<size_t>(s.g) * k;
    double* sd = pf + static_cast<size_t>(s.g) * k * d;
    if (ng == 0) {   // an empty shard contributes identity partials
      ckc(cudaSetDevice(primary_), "cudaSetDevice");
      ckc(cudaMemsetAsync(cd, 0, static_cast<size_t>(k) * 8, lst_), "cudaMemsetAsync");
      ckc(cudaMemsetAsync(sd, 0, static_cast<size_t>(k) * d * 8, lst_), "cudaMemsetAsync");
      return;
    }
    int32_t* ad = static_cast<int32_t*>(assign->p) + s.lo;
    auto* cg = static_cast<int64_t*>(shard_buf(s, cd, static_cast<size_t>(k) * 8));
    auto* sg = static_cast<double*>(shard_buf(s, sd, static_cast<size_t>(k) * d * 8));
    auto* ag = static_cast<int32_t*>(shard_buf(s, ad, static_cast<size_t>(ng) * 4));
    const auto* xw = static_cast<const double*>(window(x, s, s.lo * d, s.hi * d));
    const auto* mw = static_cast<const double*>(window(mu, s, 0, static_cast<int64_t>(k) * d));
    const size_t wsb = dlx_kmeans_workspace_bytes(ng, d, k);
    void* ws = nullptr;
    ckc(cudaMallocAsync(&ws, std::max<size_t>(16, wsb), s.st), "cudaMallocAsync");
    const int rc = dlx_kmeans_step(xw, ng, d, k, mw, ag, cg, sg, ws, wsb, DLX_KMEANS_AUTO, s.st);
    cudaFreeAsync(ws, s.st);
    ck(rc);
    copy_back(s, cd, primary_, cg, static_cast<size_t>(k) * 8);
    copy_back(s, sd, primary_, sg, static_cast<size_t>(k) * d * 8);
    copy_back(s, ad, primary_, ag, static_cast<size_t>(ng) * 4);
  });
  // ascending-shard fold (fused with the centroid update when the group targets mu itself)
  auto* counts = static_cast<int64_t*>(dalloc(static_cast<size_t>(k) * 8));
  auto* sums = static_cast<double*>(dalloc(static_cast<size_t>(k) * d * 8));
  int rc;
  if (U && U == mu) {
    rc = combine_kmeans_update(pf, sums, reinterpret_cast<const long long*>(pi), reinterpret_cast<long long*>(counts), k,
                               d, G, static_cast<double*>(U->p), lst_);
  } else {
    rc = combine_f64_i64(pf, static_cast<long long>(k) * d, sums, reinterpret_cast<const long long*>(pi), k,
                         reinterpret_cast<long long*>(counts), G, lst_);
    if (rc == DLX_OK && U) rc = dlx_kmeans_update(counts, sums, k, d, static_cast<double*>(U->p), lst_);
  }
  const bool copy_sums = !U || !p.sums_group_only;
  int64_t* hres = res_->pin.get_n<int64_t>(p.nres);
  if (rc == DLX_OK) {
    cudaMemcpyAsync(hres, counts, static_cast<size_t>(k) * 8, cudaMemcpyDeviceToHost, lst_);
    if (copy_sums) cudaMemcpyAsync(hres + k, sums, static_cast<size_t>(k) * d * 8, cudaMemcpyDeviceToHost, lst_);
  }
  dfree(pi);
  dfree(pf);
  dfree(counts);
  dfree(sums);
  ck(rc);
  cudaEvent_t ev = complete_loop({}, nullptr);
  assign->wev = ev;
  for (const LoopPlan::Out& o : p.outs) {
    if (o.src == 1) bind(o.sym, Val{assign});
    else if (!(U && o.group_only)) bind(o.sym, Val{make_lazy(hres + o.ix, o.ty, 8)});
  }
  if (U) {
    U->wev = ev;
    U->host_valid = false;
    U->page_valid = false;
    U->touched();
    for (int q : p.skip) mark_skip(q);
  }
  rep["update"] = U ? "device" : p.upd_vec >= 0 ? "host" : "none";
}

void Executor::launch_groupby_sharded(LoopPlan& p, int64_t n, std::vector<VecP>& V) {
  const VecP& keys = V[p.keys];
  if (n > keys->n) load_trap();
  wait_inputs(V);
  const int64_t K = p.k;
  std::vector<Shard> sh = shards(n);
  const int G = static_cast<int>(sh.size());
  auto* pi = static_cast<int64_t*>(dalloc(static_cast<size_t>(G) * K * 8));
  run_shards(sh, [&](Shard& s) {
    const int64_t ng = s.hi - s.lo;
    int64_t* cd = pi + static_cast<size_t>(s.g) * K;
    if (ng == 0) {
      ckc(cudaSetDevice(primary_), "cudaSetDevice");
      ckc(cudaMemsetAsync(cd, 0, static_cast<size_t>(K) * 8, lst_), "cudaMemsetAsync");
      return;
    }
    auto* cg = static_cast<int64_t*>(shard_buf(s, cd, static_cast<size_t>(K) * 8));
    const auto* kw = static_cast<const int64_t*>(window(keys, s, s.lo, s.hi));
    const size_t wsb = dlx_groupby_workspace_bytes(ng, K);
    void* ws = nullptr;
    ckc(cudaMallocAsync(&ws, std::max<size_t>(16, wsb), s.st), "cudaMallocAsync");
    const int rc = dlx_groupby_count(kw, ng, K, cg, ws, wsb, s.st);
    cudaFreeAsync(ws, s.st);
    ck(rc);
    copy_back(s, cd, primary_, cg, static_cast<size_t>(K) * 8);
  });
  auto* counts = static_cast<int64_t*>(dalloc(static_cast<size_t>(K) * 8));
  int rc = combine_f64_i64(nullptr, 0, nullptr, reinterpret_cast<const long long*>(pi), K,
                           reinterpret_cast<long long*>(counts), G, lst_);
  int64_t* hres = res_->pin.get_n<int64_t>(K);
  if (rc == DLX_OK) cudaMemcpyAsync(hres, counts, static_cast<size_t>(K) * 8, cudaMemcpyDeviceToHost, lst_);
  dfree(pi);
  dfree(counts);
  ck(rc);
  complete_loop({}, nullptr);
  bind_scalars(p, hres);
}

void Executor::launch_bucket_rows_sharded(LoopPlan& p, int64_t n, std::vector<VecP>& V) {
  const VecP& x = V[p.x];
  const VecP& keys = V[p.keys];
  if (n > keys->n || n * p.d > x->n) load_trap();
  wait_inputs(V);
  const int32_t d = static_cast<int32_t>(p.d), K = static_cast<int32_t>(p.k);
  std::vector<Shard> sh = shards(n);
  const int G = static_cast<int>(sh.size());
  auto* pi = static_cast<int64_t*>(dalloc(static_cast<size_t>(G) * K * 8));
  auto* pf = static_cast<double*>(dalloc(static_cast<size_t>(G) * K * d * 8));
  run_shards(sh, [&](Shard& s) {
    const int64_t ng = s.hi - s.lo;
    int64_t* cd = pi + static_cast<size_t>(s.g) * K;
    double* sd = pf + static_cast<size_t>(s.g) * K * d;
    if (ng == 0) {
      ckc(cudaSetDevice(primary_), "cudaSetDevice");
      ckc(cudaMemsetAsync(cd, 0, static_cast<size_t>(K) * 8, lst_), "cudaMemsetAsync");
      ckc(cudaMemsetAsync(sd, 0, static_cast<size_t>(K) * d * 8, lst_), "cudaMemsetAsync");
      return;
    }
    auto* cg = static_cast<int64_t*>(shard_buf(s, cd, static_cast<size_t>(K) * 8));
    auto* sg = static_cast<double*>(shard_buf(s, sd, static_cast<size_t>(K) * d * 8));
    const auto* xw = static_cast<const double*>(window(x, s, s.lo * d, s.hi * d));
    const auto* kw = static_cast<const int64_t*>(window(keys, s, s.lo, s.hi));
    const size_t wsb = dlx_bucket_rowsum_workspace_bytes(ng, d, K);
    void* ws = nullptr;
    ckc(cudaMallocAsync(&ws, std::max<size_t>(16, wsb), s.st), "cudaMallocAsync");
    const int rc = dlx_bucket_rowsum(xw, kw, ng, d, p.buckets.data(), K, cg, sg, ws, wsb, s.st);
    cudaFreeAsync(ws, s.st);
    ck(rc);
    copy_back(s, cd, primary_, cg, static_cast<size_t>(K) * 8);
    copy_back(s, sd, primary_, sg, static_cast<size_t>(K) * d * 8);
  });
  auto* rec = static_cast<int64_t*>(dalloc(p.nres * 8));   // counts[K], then sums[K][d]
  int rc = combine_f64_i64(pf, static_cast<long long>(K) * d, reinterpret_cast<double*>(rec + K),
                           reinterpret_cast<const long long*>(pi), K, reinterpret_cast<long long*>(rec), G, lst_);
  int64_t* hres = res_->pin.get_n<int64_t>(p.nres);
  if (rc == DLX_OK) cudaMemcpyAsync(hres, rec, p.nres * 8, cudaMemcpyDeviceToHost, lst_);
  dfree(pi);
  dfree(pf);
  dfree(rec);
  ck(rc);
  complete_loop({}, nullptr);
  bind_scalars(p, hres);
}

void Executor::launch_gda2_sharded(LoopPlan& p, int64_t n, std::vector<VecP>& V) {
  const VecP& X = V[p.x];
  const VecP& Y = V[p.keys];
  const int64_t d = p.d;
  if (n * d > X->n || n > Y->n) load_trap();
  double* hmu = res_->pin.get_n<double>(2 * d);
  for (int64_t c = 0; c < d; ++c) {
    hmu[c] = p.m0sym[c] >= 0 ? force(env_[p.m0sym[c]]).d() : p.m0lit[c];
    hmu[d + c] = p.m1sym[c] >= 0 ? force(env_[p.m1sym[c]]).d() : p.m1lit[c];
  }
  wait_inputs(V);
  std::vector<Shard> sh = shards(n);
  const int G = static_cast<int>(sh.size());
  auto* pf = static_cast<double*>(dalloc(static_cast<size_t>(G) * d * d * 8));
  run_shards(sh, [&](Shard& s) {
    const int64_t ng = s.hi - s.lo;
    double* sd = pf + static_cast<size_t>(s.g) * d * d;
    if (ng == 0) {
      ckc(cudaSetDevice(primary_), "cudaSetDevice");
      ckc(cudaMemsetAsync(sd, 0, static_cast<size_t>(d) * d * 8, lst_), "cudaMemsetAsync");
      return;
    }
    auto* sg = static_cast<double*>(shard_buf(s, sd, static_cast<size_t>(d) * d * 8));
    const auto* xw = static_cast<const double*>(window(X, s, s.lo * d, s.hi * d));
    const auto* yw = static_cast<const int64_t*>(window(Y, s, s.lo, s.hi));
    const size_t wsb = dlx_gda_workspace_bytes(ng, static_cast<int32_t>(d));
    void* ws = nullptr;
    double* dmu = nullptr;
    ckc(cudaMallocAsync(&ws, std::max<size_t>(16, wsb), s.st), "cudaMallocAsync");
    ckc(cudaMallocAsync(&dmu, 2 * d * 8, s.st), "cudaMallocAsync");
    ckc(cudaMemcpyAsync(dmu, hmu, 2 * d * 8, cudaMemcpyHostToDevice, s.st), "h2d means");
    const int rc = dlx_gda_pass2(xw, yw, ng, static_cast<int32_t>(d), dmu, dmu + d, sg, ws, wsb, s.st);
    cudaFreeAsync(ws, s.st);
    cudaFreeAsync(dmu, s.st);
    ck(rc);
    copy_back(s, sd, primary_, sg, static_cast<size_t>(d) * d * 8);
  });
  auto* S = static_cast<double*>(dalloc(d * d * 8));
  int rc = combine_f64(pf, G, d * d, S, lst_);
  int64_t* hres = res_->pin.get_n<int64_t>(d * d);
  if (rc == DLX_OK) cudaMemcpyAsync(hres, S, d * d * 8, cudaMemcpyDeviceToHost, lst_);
  dfree(pf);
  dfree(S);
  ck(rc);
  complete_loop({}, nullptr);
  bind_scalars(p, hres);
}

void Executor::launch_logistic_sharded(LoopPlan& p, int64_t n, std::vector<VecP>& V, nlohmann::json& rep) {
  const VecP& X = V[p.x];
  const VecP& TH = V[p.mu];
  const VecP& Y = V[p.keys];
  const int32_t d = static_cast<int32_t>(p.d);
  if (n * d > X->n || d > TH->n || n > Y->n) load_trap();
  dlx_link_code link = p.link;
  for (auto [q, sym] : p.link_patches) link.imm[q] = force(env_[sym]).d();
  double alpha = p.alpha_lit;
  VecP U;
  if (p.upd_vec >= 0 && bound_[p.upd_vec] && env_[p.upd_vec].is_vec()) {
    U = env_[p.upd_vec].vec();
    if (U->elem != Ty::Double || U->n != d) U = nullptr;
    if (U && p.alpha_sym >= 0) {
      Val a = force(env_[p.alpha_sym]);
      if (a.is_dbl()) alpha = a.d();
      else U = nullptr;
    }
  }
  wait_inputs(V);
  if (U) {
    fence_on(lst_);
    if (U->wev) cudaStreamWaitEvent(lst_, U->wev, 0);
  }
  std::vector<Shard> sh = shards(n);
  const int G = static_cast<int>(sh.size());
  VecP h = new_vec(n, Ty::Double, lst_, false);
  auto* pf = static_cast<double*>(dalloc(static_cast<size_t>(G) * d * 8));
  run_shards(sh, [&](Shard& s) {
    const int64_t ng = s.hi - s.lo;
    double* gd = pf + static_cast<size_t>(s.g) * d;
    if (ng == 0) {
      ckc(cudaSetDevice(primary_), "cudaSetDevice");
      ckc(cudaMemsetAsync(gd, 0, static_cast<size_t>(d) * 8, lst_), "cudaMemsetAsync");
      return;
    }
    double* hd = static_cast<double*>(h->p) + s.lo;
    auto* gg = static_cast<double*>(shard_buf(s, gd, static_cast<size_t>(d) * 8));
    auto* hg = static_cast<double*>(shard_buf(s, hd, static_cast<size_t>(ng) * 8));
    const auto* xw = static_cast<const double*>(window(X, s, s.lo * d, s.hi * d));
    const auto* yw = static_cast<const int64_t*>(window(Y, s, s.lo, s.hi));
    const auto* tw = static_cast<const double*>(window(TH, s, 0, d));
    const size_t wsb = dlx_logreg_workspace_bytes(ng, d);
    void* ws = nullptr;
    ckc(cudaMallocAsync(&ws, std::max<size_t>(16, wsb), s.st), "cudaMallocAsync");
    const int rc = dlx_rowdot_link_grad(xw, yw, ng, d, tw, &link, hg, gg, ws, wsb, s.st);
    cudaFreeAsync(ws, s.st);
    ck(rc);
    copy_back(s, gd, primary_, gg, static_cast<size_t>(d) * 8);
    copy_back(s, hd, primary_, hg, static_cast<size_t>(ng) * 8);
  });
  auto* grad = static_cast<double*>(dalloc(static_cast<size_t>(d) * 8));
  int rc = combine_f64(pf, G, d, grad, lst_);
  if (rc == DLX_OK && U) rc = dlx_axpy_inplace(static_cast<double*>(U->p), grad, alpha, d, lst_);
  const bool copy_grad = !U || !p.sums_group_only;
  int64_t* hres = res_->pin.get_n<int64_t>(d);
  if (rc == DLX_OK && copy_grad) cudaMemcpyAsync(hres, grad, static_cast<size_t>(d) * 8, cudaMemcpyDeviceToHost, lst_);
  dfree(pf);
  dfree(grad);
  ck(rc);
  cudaEvent_t ev = complete_loop({}, nullptr);
  h->wev = ev;
  for (const LoopPlan::Out& o : p.outs) {
    if (o.src == 1) bind(o.sym, Val{h});
    else if (!(U && o.group_only)) bind(o.sym, Val{make_lazy(hres + o.ix, o.ty, 8)});
  }
  if (U) {
    U->wev = ev;
    U->host_valid = false;
    U->page_valid = false;
    U->touched();
    for (int q : p.skip) mark_skip(q);
  }
  rep["update"] = U ? "device" : p.upd_vec >= 0 ? "host" : "none";
}

}  // namespace dlx
