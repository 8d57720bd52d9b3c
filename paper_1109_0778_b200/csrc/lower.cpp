// lower.cpp — the CUDA target's ParallelLoop handler (the B200 replacement of
// emit_parallel_loop, proj/src/codegen.cpp:345-433): every live elem of a root loop is
// symbolically evaluated into an expression DAG (loads at affine indices, scalar ops, nested
// reduces, the reduce `combine` block recognised as + / * of rv_left / rv_right), then matched
// against the specialised families and lowered to their kernels:
//   kmeans       argmin chain over k nested distance reduces + k counts and k*d sums keyed on
//                it (a4)                                 -> dlx_kmeans_step / _iteration
//   groupby      K count reduces keyed on key(i) == b (a7)  -> dlx_groupby_count
//   bucket_rows  counts and column sums keyed on key(i) == b (GDA pass 1, a6) -> dlx_bucket_rowsum
//   gda_scatter  d*d centred products with per-class mean selects (GDA pass 2, a6) -> dlx_gda_pass2
//   generic      anything else within the generic kernel's plan (vm.cu)  -> dlx_vm_run_loop
// Loops none of them can lower raise GenerationFailed (codegen.cpp:66-71) — no CPU fallback.
// The result of a lowering (LoopPlan) is cached per loop statement in the program, so a
// program executed again (or a While body) skips the symbolic evaluation.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <tuple>

#include "program_exec.hpp"

namespace dlx {

using json = nlohmann::json;

#define MISS(why)                                                                     \
  do {                                                                                \
    if (g_run->debug) fprintf(stderr, "[dlx program] %s: %s\n", __func__, why);       \
    return false;                                                                     \
  } while (0)

namespace {
SEP mk(SE::K k, Ty ty) {
  auto s = std::make_shared<SE>();
  s->k = k;
  s->ty = ty;
  return s;
}
int64_t val_bits(const Val& v) {
  if (v.is_int()) return v.i();
  if (v.is_bool()) return v.b();
  if (v.is_dbl()) {
    int64_t b;
    double d = v.d();
    std::memcpy(&b, &d, 8);
    return b;
  }
  return 0;
}
// the same value: one node, or two literal nodes with equal payloads (literals are not shared)
bool same_se(const SEP& x, const SEP& y) {
  if (x == y) return true;
  if (x->k == SE::Const && y->k == SE::Const && x->ty == y->ty)
    return x->ty == Ty::Double ? std::memcmp(&x->cd, &y->cd, 8) == 0 : x->ci == y->ci;
  return false;
}
bool is_rv_pair(const SEP& c, Op op) {
  return c->k == SE::Bin && c->op == op &&
         ((c->a[0]->k == SE::RvL && c->a[1]->k == SE::RvR) || (c->a[0]->k == SE::RvR && c->a[1]->k == SE::RvL));
}
bool is_plus_combine(const SEP& c) { return is_rv_pair(c, Op::Plus); }
bool is_times_combine(const SEP& c) { return is_rv_pair(c, Op::Times); }
bool zero_is(const Atom& z, int64_t iv) { return z.k == Atom::Int && z.i == iv; }
bool zero_is_pos0(const Atom& z) {
  if (z.k != Atom::Double) return false;
  const double pz = 0.0;
  return std::memcmp(&z.d, &pz, 8) == 0;
}
}  // namespace

int MatchCtx::slot(const SEP& vn) {
  for (size_t q = 0; q < vsyms.size(); ++q)
    if (vsyms[q] == vn->sym) return static_cast<int>(q);
  vsyms.push_back(vn->sym);
  vecs.push_back(vn->vec);
  return static_cast<int>(vsyms.size()) - 1;
}
void MatchCtx::bake(const SEP& s) {
  if (s->k == SE::Host) baked.emplace_back(s->sym, val_bits(s->host));
}

bool Executor::is_const_int(const SEP& s, int64_t* v) {
  if (s->k == SE::Const && s->ty == Ty::Int) {
    if (v) *v = s->ci;
    return true;
  }
  if (s->k == SE::Host && s->host.is_int()) {
    if (v) *v = s->host.i();
    if (mc_) mc_->bake(s);
    return true;
  }
  return false;
}
bool Executor::is_const_dbl(const SEP& s, double* v) {
  if (s->k == SE::Const && s->ty == Ty::Double) {
    if (v) *v = s->cd;
    return true;
  }
  if (s->k == SE::Host && s->host.is_dbl()) {
    if (v) *v = s->host.d();
    if (mc_) mc_->bake(s);
    return true;
  }
  return false;
}

// affine form a*Idx + b*Inner(sym) + c
bool Executor::affine(const SEP& s, Affine* out) {
  int64_t v;
  if (is_const_int(s, &v)) return *out = Affine{0, 0, v, -1}, true;
  if (s->k == SE::Idx) return *out = Affine{1, 0, 0, -1}, true;
  if (s->k == SE::Inner) return *out = Affine{0, 1, 0, s->sym}, true;
  if (s->k == SE::Bin && (s->op == Op::Plus || s->op == Op::Minus || s->op == Op::Times)) {
    Affine x, y;
    if (!affine(s->a[0], &x) || !affine(s->a[1], &y)) return false;
    if (x.inner >= 0 && y.inner >= 0 && x.inner != y.inner) return false;
    const int inner = x.inner >= 0 ? x.inner : y.inner;
    if (s->op == Op::Plus) return *out = Affine{x.a + y.a, x.b + y.b, x.c + y.c, inner}, true;
    if (s->op == Op::Minus) return *out = Affine{x.a - y.a, x.b - y.b, x.c - y.c, inner}, true;
    if (x.a == 0 && x.b == 0) return *out = Affine{x.c * y.a, x.c * y.b, x.c * y.c, inner}, true;
    if (y.a == 0 && y.b == 0) return *out = Affine{y.c * x.a, y.c * x.b, y.c * x.c, inner}, true;
  }
  return false;
}

// ---- symbolic evaluation of a loop body ------------------------------------------------------
SEP Executor::sym_atom(const Atom& a) {
  switch (a.k) {
    case Atom::Sym: {
      if (a.sym == loop_index_) return mk(SE::Idx, Ty::Int);
      auto it = sym_.find(a.sym);
      if (it != sym_.end()) return it->second;
      if (a.sym < 0 || a.sym > P.max_sym) gen_fail("loop body reads x" + std::to_string(a.sym) + ", not a program symbol");
      if (!bound_[a.sym] && !pending_.empty()) join_all();
      if (!bound_[a.sym]) gen_fail("loop body reads x" + std::to_string(a.sym) + " before definition");
      mc_->deps.push_back(a.sym);
      Val v = env_[a.sym];
      SEP s;
      if (v.is_vec()) {
        s = mk(SE::Vec, v.vec()->elem);
        s->vec = v.vec();
      } else {
        v = force(v);
        if (!v.is_int() && !v.is_dbl() && !v.is_bool()) gen_fail("loop body reads a non-scalar host value");
        s = mk(SE::Host, v.is_int() ? Ty::Int : v.is_dbl() ? Ty::Double : Ty::Bool);
        s->host = v;
      }
      s->sym = a.sym;
      sym_[a.sym] = s;   // one node per env symbol
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
    case Atom::Unit: return mk(SE::Const, Ty::Unit);   // body-scope results are Unit
    default: gen_fail("non-scalar constant in a loop body");
  }
}

SEP Executor::sym_block(int b) {
  const Block& bl = P.block(b);
  for (int s : bl.stmts) sym_[s] = sym_stmt(P.stmts[s]);
  return sym_atom(bl.result);
}

SEP Executor::sym_stmt(const Stmt& s) {
  const Ty ty = s.ty.t;
  switch (s.op) {
    case Op::Plus: case Op::Minus: case Op::Times: case Op::Divide: case Op::Lt: case Op::Eq:
    case Op::And: case Op::Or: {
      auto e = mk(SE::Bin, ty);
      e->op = s.op;
      e->a = {sym_atom(s.args[0]), sym_atom(s.args[1])};
      return e;
    }
    case Op::Not: case Op::MathAbs: case Op::MathSqrt: case Op::ToDouble: case Op::MathExp: {
      auto e = mk(SE::Un, ty);
      e->op = s.op;
      e->a = {sym_atom(s.args[0])};
      return e;
    }
    case Op::IfThenElse: {
      auto c = sym_atom(s.args[0]);
      auto t = sym_block(s.blocks[0]);
      auto f = sym_block(s.blocks[1]);
      auto e = mk(SE::Sel, ty);
      e->a = {c, t, f};
      return e;
    }
    case Op::VectorApply: {
      auto e = mk(SE::Load, ty);
      e->a = {sym_atom(s.args[0]), sym_atom(s.args[1])};
      if (e->a[0]->k != SE::Vec) gen_fail("element load from a vector produced inside the loop");
      return e;
    }
    case Op::VectorLength: {
      auto v = sym_atom(s.args[0]);
      if (v->k != SE::Vec) gen_fail("length of a loop-local vector");
      auto e = mk(SE::Const, Ty::Int);
      e->ci = v->vec->n;
      return e;
    }
    case Op::ParallelLoop: {
      // nested (possibly horizontally fused) loop: every live elem must be a plain reduce over a
      // loop-invariant range; each becomes one Red node bound to its elem's `out`
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
        if (e.kind != Elem::Reduce || e.cond >= 0) gen_fail("nested loop elem other than a plain reduce");
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
    default: break;
  }
  gen_fail("don't know how to generate code for: " + s.opname + " inside a multiloop");
}

// ---- family: fused k-means (argmin collect + bucket counts / sums keyed on it) ----------------
// D = Red(range d, zero 0.0, Plus, Times(t, t), t = Load(X, d*Idx + J) - Load(M, c*d + J))
bool Executor::match_distance(const SEP& D, int64_t c, LoopPlan& p, MatchCtx& m) {
  if (D->k != SE::Red || D->ty != Ty::Double || !is_plus_combine(D->a[1])) MISS("not a + reduce");
  if (!zero_is_pos0(D->zero)) MISS("zero is not 0.0");
  const SEP& el = D->a[0];
  if (el->k != SE::Bin || el->op != Op::Times || !same_se(el->a[0], el->a[1])) MISS("not a square");
  const SEP& t = el->a[0];
  if (t->k != SE::Bin || t->op != Op::Minus || t->a[0]->k != SE::Load || t->a[1]->k != SE::Load) MISS("not a difference of loads");
  Affine ax, am;
  if (!affine(t->a[0]->a[1], &ax) || !affine(t->a[1]->a[1], &am)) MISS("non-affine index");
  const int64_t d = D->range;
  if (ax.a != d || ax.b != 1 || ax.c != 0 || ax.inner != D->sym) MISS("x index is not d*i + j");
  if (am.a != 0 || am.b != 1 || am.c != c * d || am.inner != D->sym) MISS("mu index is not c*d + j");
  if (t->a[0]->a[0]->ty != Ty::Double || t->a[1]->a[0]->ty != Ty::Double) MISS("not Double vectors");
  const int xs = m.slot(t->a[0]->a[0]), ms = m.slot(t->a[1]->a[0]);
  if (p.x >= 0 && (p.x != xs || p.mu != ms || p.d != d)) MISS("different x / mu / d across centroids");
  p.x = xs;
  p.mu = ms;
  p.d = d;
  return true;
}

// chain: idx_{c+1} = Sel(lt_c, c, idx_c), best_{c+1} = Sel(lt_c, D_c, best_c),
// lt_c = Lt(D_c, best_c), idx_0 = 0, best_0 = 1e300 (staged_if chain, stage.cpp:73-104)
bool Executor::match_argmin(const SEP& root, LoopPlan& p, MatchCtx& m) {
  std::vector<SEP> levels;
  SEP cur = root;
  while (cur->k == SE::Sel && cur->ty == Ty::Int) {
    levels.push_back(cur);
    cur = cur->a[2];
  }
  int64_t z;
  if (!is_const_int(cur, &z) || z != 0 || levels.empty()) MISS("chain does not start at index 0");
  const int64_t k = static_cast<int64_t>(levels.size());
  SEP best_prev;
  for (int64_t c = 0; c < k; ++c) {
    const SEP& lv = levels[k - 1 - c];
    int64_t cv;
    if (!is_const_int(lv->a[1], &cv) || cv != c) MISS("level index is not c");
    const SEP& lt = lv->a[0];
    if (lt->k != SE::Bin || lt->op != Op::Lt) MISS("level condition is not <");
    const SEP& D = lt->a[0];
    const SEP& B = lt->a[1];
    if (c == 0) {
      double bd;
      if (!is_const_dbl(B, &bd) || bd != 1e300) MISS("chain does not start at 1e300");
    } else if (!same_se(B, best_prev)) {
      MISS("level compares against another best");
    }
    if (!match_distance(D, c, p, m)) MISS("distance");
    best_prev = nullptr;
    if (c + 1 < k) {
      const SEP& nlt = levels[k - 2 - c]->a[0];
      if (nlt->k != SE::Bin || nlt->op != Op::Lt) MISS("next level condition is not <");
      const SEP& nB = nlt->a[1];
      if (nB->k != SE::Sel || !same_se(nB->a[0], lt) || !same_se(nB->a[1], D) || !same_se(nB->a[2], B))
        MISS("best is not Sel(lt, D, best)");
      best_prev = nB;
    }
  }
  p.k = k;
  return true;
}

bool Executor::match_kmeans(const Stmt& s, int64_t n, std::vector<LElem>& els, LoopPlan& p, MatchCtx& m) {
  (void)n;
  int ci = -1;
  for (size_t q = 0; q < els.size(); ++q)
    if (els[q].e->kind == Elem::Collect) {
      if (ci >= 0) MISS("two collects");
      ci = static_cast<int>(q);
    }
  if (ci < 0 || els[ci].cond || els[ci].e->append) MISS("no dense collect");
  p.x = p.mu = -1;
  p.d = p.k = 0;
  if (!match_argmin(els[ci].value, p, m)) MISS("argmin");
  const SEP key = els[ci].value;
  const int64_t d = p.d, k = p.k;
  p.outs.clear();
  std::unordered_map<int, std::tuple<int, int64_t, int64_t>> slot_of;   // out -> (0 count / 1 sum, c, j)
  for (size_t q = 0; q < els.size(); ++q) {
    const LElem& le = els[q];
    if (static_cast<int>(q) == ci) {
      p.outs.push_back({le.e->out, 1, 0, Ty::Int});
      continue;
    }
    if (le.e->kind != Elem::Reduce || !le.cond || !is_plus_combine(le.combine)) MISS("elem is not a keyed + reduce");
    const SEP& cd = le.cond;
    if (cd->k != SE::Bin || cd->op != Op::Eq) MISS("cond is not ==");
    int64_t c;
    if (cd->a[0] == key && is_const_int(cd->a[1], &c)) {
    } else if (cd->a[1] == key && is_const_int(cd->a[0], &c)) {
    } else {
      MISS("cond is not assign == c");
    }
    if (c < 0 || c >= k) MISS("bucket outside [0, k)");
    int64_t one;
    if (is_const_int(le.value, &one) && one == 1 && zero_is(le.e->zero, 0)) {
      p.outs.push_back({le.e->out, 0, c, Ty::Int});
      slot_of[le.e->out] = {0, c, 0};
    } else if (le.value->k == SE::Load && le.value->a[0]->k == SE::Vec && m.slot(le.value->a[0]) == p.x &&
               zero_is_pos0(le.e->zero)) {
      Affine af;
      if (!affine(le.value->a[1], &af) || af.a != d || af.b != 0 || af.c < 0 || af.c >= d) MISS("sum index is not d*i + j");
      p.outs.push_back({le.e->out, 0, k + c * d + af.c, Ty::Double});
      slot_of[le.e->out] = {1, c, af.c};
    } else {
      MISS("elem is neither a count nor a column sum");
    }
  }
  p.nres = k + k * d;
  // the centroid update after the loop (UpdateGroup): on the device when its k*d updates are
  // exactly mu(c*d + j) = sum_cj / toDouble(count_c)
  p.upd_vec = -1;
  p.skip.clear();
  p.sums_group_only = false;
  auto g = P.update_after.find(s.sym);
  if (g != P.update_after.end() && g->second.kind == UpdateGroup::Div &&
      static_cast<int64_t>(g->second.entries.size()) == k * d) {
    std::vector<uint8_t> seen(k * d, 0);
    bool ok = true;
    for (const UpdateGroup::Entry& en : g->second.entries) {
      auto cs = slot_of.find(en.count_sym), ss = slot_of.find(en.sum_sym);
      if (cs == slot_of.end() || ss == slot_of.end() || std::get<0>(cs->second) != 0 || std::get<0>(ss->second) != 1 ||
          std::get<1>(cs->second) != std::get<1>(ss->second) ||
          en.e != std::get<1>(ss->second) * d + std::get<2>(ss->second) || en.e < 0 || en.e >= k * d || seen[en.e]) {
        ok = false;
        break;
      }
      seen[en.e] = 1;
    }
    if (ok) {
      p.upd_vec = g->second.vec_sym;
      p.skip = g->second.stmts;
      std::unordered_map<int, int> group_reads;   // sum -> reads by the group's divides
      for (const UpdateGroup::Entry& en : g->second.entries) ++group_reads[en.sum_sym];
      size_t only = 0;
      for (LoopPlan::Out& o : p.outs) {
        auto it = group_reads.find(o.sym);
        o.group_only = it != group_reads.end() && P.uses[o.sym] == it->second;
        only += o.group_only;
      }
      p.sums_group_only = only == static_cast<size_t>(k * d);
    } else if (g_run->debug) {
      fprintf(stderr, "[dlx program] update group after x%d does not cover mu(c*d+j) = sum/count\n", s.sym);
    }
  }
  p.fam = LoopPlan::Kmeans;
  p.family = "kmeans";
  p.launch = p.upd_vec >= 0 ? "dlx_kmeans_iteration" : "dlx_kmeans_step";
  return true;
}

// ---- family: bucket counts (GroupBy) ------------------------------------------------------
bool Executor::match_groupby(int64_t n, std::vector<LElem>& els, LoopPlan& p, MatchCtx& m) {
  (void)n;
  int ks = -1;
  int64_t nb = 0;
  p.outs.clear();
  for (const LElem& le : els) {
    int64_t one;
    if (le.e->kind != Elem::Reduce || !le.cond || !is_plus_combine(le.combine) || !is_const_int(le.value, &one) ||
        one != 1 || !zero_is(le.e->zero, 0))
      MISS("elem is not a keyed count");
    const SEP& cd = le.cond;
    if (cd->k != SE::Bin || cd->op != Op::Eq) MISS("cond is not ==");
    SEP ld = cd->a[0], cs = cd->a[1];
    if (ld->k != SE::Load) std::swap(ld, cs);
    int64_t b;
    if (ld->k != SE::Load || !is_const_int(cs, &b) || b < 0) MISS("cond is not key(i) == b");
    Affine af;
    if (!affine(ld->a[1], &af) || af.a != 1 || af.b != 0 || af.c != 0 || ld->a[0]->ty != Ty::Int) MISS("key index is not i");
    const int s = m.slot(ld->a[0]);
    if (ks >= 0 && ks != s) MISS("two key vectors");
    ks = s;
    p.outs.push_back({le.e->out, 0, b, Ty::Int});
    nb = std::max(nb, b + 1);
  }
  if (ks < 0 || nb > (1 << 24)) MISS("no keys / too many buckets");
  p.keys = ks;
  p.k = nb;
  p.nres = nb;
  p.fam = LoopPlan::GroupBy;
  p.family = "groupby";
  p.launch = "dlx_groupby_count";
  return true;
}

// ---- family: bucket row sums (GDA pass 1: a count and d column sums per class) -----------------
// every elem: cond Eq(Load(Y, i), b); value 1 (count, zero 0) or Load(X, d*i + j) (zero 0.0)
bool Executor::match_bucket_rows(int64_t n, std::vector<LElem>& els, LoopPlan& p, MatchCtx& m) {
  (void)n;
  int ys = -1;
  p.x = -1;
  p.d = 0;
  p.buckets.clear();
  struct E { int out; int64_t b; int64_t j; bool sum; };
  std::vector<E> es;
  bool any_sum = false;
  for (const LElem& le : els) {
    if (le.e->kind != Elem::Reduce || !le.cond || !is_plus_combine(le.combine)) MISS("elem is not a keyed + reduce");
    const SEP& cd = le.cond;
    if (cd->k != SE::Bin || cd->op != Op::Eq) MISS("cond is not ==");
    SEP ld = cd->a[0], cs = cd->a[1];
    if (ld->k != SE::Load) std::swap(ld, cs);
    int64_t b;
    if (ld->k != SE::Load || !is_const_int(cs, &b)) MISS("cond is not key(i) == b");
    Affine ay;
    if (!affine(ld->a[1], &ay) || ay.a != 1 || ay.b != 0 || ay.c != 0 || ld->a[0]->ty != Ty::Int) MISS("key index is not i");
    const int s = m.slot(ld->a[0]);
    if (ys >= 0 && ys != s) MISS("two key vectors");
    ys = s;
    int64_t one;
    if (is_const_int(le.value, &one) && one == 1 && zero_is(le.e->zero, 0)) {
      es.push_back({le.e->out, b, 0, false});
    } else if (le.value->k == SE::Load && le.value->a[0]->ty == Ty::Double && zero_is_pos0(le.e->zero)) {
      Affine ax;
      if (!affine(le.value->a[1], &ax) || ax.b != 0 || ax.a <= 0 || ax.c < 0 || ax.c >= ax.a) MISS("sum index is not d*i + j");
      const int xs = m.slot(le.value->a[0]);
      if ((p.x >= 0 && p.x != xs) || (p.d && p.d != ax.a)) MISS("two row layouts");
      p.x = xs;
      p.d = ax.a;
      es.push_back({le.e->out, b, ax.c, true});
      any_sum = true;
    } else {
      MISS("elem is neither a count nor a column sum");
    }
  }
  if (!any_sum || ys < 0) MISS("no column sums");
  for (const E& e : es)
    if (std::find(p.buckets.begin(), p.buckets.end(), e.b) == p.buckets.end()) p.buckets.push_back(e.b);
  if (p.buckets.size() > 64 || p.d > 256) MISS("too many buckets / columns");
  const int64_t K = static_cast<int64_t>(p.buckets.size());
  p.outs.clear();
  for (const E& e : es) {
    const int64_t t = std::find(p.buckets.begin(), p.buckets.end(), e.b) - p.buckets.begin();
    p.outs.push_back({e.out, 0, e.sum ? K + t * p.d + e.j : t, e.sum ? Ty::Double : Ty::Int});
  }
  p.keys = ys;
  p.k = K;
  p.nres = K + K * p.d;
  p.fam = LoopPlan::BucketRows;
  p.family = "bucket_rows";
  p.launch = "dlx_bucket_rowsum";
  return true;
}

// ---- family: GDA pass 2 (d*d scatter with per-class mean select) -------------------------------
// value = Times(Minus(Load(X, d*Idx + a), Sel_a), Minus(Load(X, d*Idx + b), Sel_b)),
// Sel = Sel(Eq(Load(Y, Idx), 1), mu1, mu0): the means are host scalars (passed per launch) or literals
bool Executor::match_centred(const SEP& t, int64_t d, int* xs, int* ys, int64_t* col, int* s0, double* l0, int* s1,
                             double* l1, MatchCtx& m) {
  if (t->k != SE::Bin || t->op != Op::Minus || t->a[0]->k != SE::Load || t->a[1]->k != SE::Sel) return false;
  Affine af;
  if (!affine(t->a[0]->a[1], &af) || af.a != d || af.b != 0 || af.c < 0 || af.c >= d) return false;
  const SEP& sel = t->a[1];
  const SEP& eq = sel->a[0];
  if (eq->k != SE::Bin || eq->op != Op::Eq) return false;
  SEP ld = eq->a[0], cs = eq->a[1];
  if (ld->k != SE::Load) std::swap(ld, cs);
  int64_t one;
  if (ld->k != SE::Load || !is_const_int(cs, &one) || one != 1) return false;
  Affine ay;
  if (!affine(ld->a[1], &ay) || ay.a != 1 || ay.b != 0 || ay.c != 0) return false;
  auto src = [](const SEP& v, int* sym, double* lit) {
    if (v->k == SE::Host && v->host.is_dbl()) return *sym = v->sym, true;
    if (v->k == SE::Const && v->ty == Ty::Double) return *sym = -1, *lit = v->cd, true;
    return false;
  };
  if (!src(sel->a[1], s1, l1) || !src(sel->a[2], s0, l0)) return false;
  if (t->a[0]->a[0]->ty != Ty::Double || ld->a[0]->ty != Ty::Int) return false;
  *xs = m.slot(t->a[0]->a[0]);
  *ys = m.slot(ld->a[0]);
  *col = af.c;
  return true;
}

bool Executor::match_gda2(int64_t n, std::vector<LElem>& els, LoopPlan& p, MatchCtx& m) {
  (void)n;
  if (els.empty()) return false;
  int64_t d = 0;
  {   // d from the first elem's row stride
    const SEP& v = els[0].value;
    if (v->k != SE::Bin || v->op != Op::Times || v->a[0]->k != SE::Bin || v->a[0]->a[0]->k != SE::Load) MISS("not a product");
    Affine af;
    if (!affine(v->a[0]->a[0]->a[1], &af)) MISS("non-affine");
    d = af.a;
  }
  if (d <= 0 || d > 128) MISS("d outside (0, 128]");
  p.m0sym.assign(d, -2);
  p.m1sym.assign(d, -2);
  p.m0lit.assign(d, 0.0);
  p.m1lit.assign(d, 0.0);
  p.cell.clear();
  p.outs.clear();
  int X = -1, Y = -1;
  for (const LElem& le : els) {
    if (le.e->kind != Elem::Reduce || le.cond || !is_plus_combine(le.combine) || !zero_is_pos0(le.e->zero))
      MISS("elem is not an unguarded + reduce from 0.0");
    const SEP& v = le.value;
    if (v->k != SE::Bin || v->op != Op::Times) MISS("not a product");
    int x1, y1, x2, y2, sa0, sa1, sb0, sb1;
    int64_t a, b;
    double la0, la1, lb0, lb1;
    if (!match_centred(v->a[0], d, &x1, &y1, &a, &sa0, &la0, &sa1, &la1, m) ||
        !match_centred(v->a[1], d, &x2, &y2, &b, &sb0, &lb0, &sb1, &lb1, m))
      MISS("factor is not x - mean(y)");
    if (x1 != x2 || y1 != y2 || (X >= 0 && (X != x1 || Y != y1))) MISS("two inputs");
    X = x1;
    Y = y1;
    for (auto [col, s0, l0, s1, l1] : {std::tuple{a, sa0, la0, sa1, la1}, std::tuple{b, sb0, lb0, sb1, lb1}}) {
      if (p.m0sym[col] != -2 && (p.m0sym[col] != s0 || p.m1sym[col] != s1 ||
                                 (s0 < 0 && p.m0lit[col] != l0) || (s1 < 0 && p.m1lit[col] != l1)))
        MISS("column mean differs across elems");
      p.m0sym[col] = s0;
      p.m1sym[col] = s1;
      p.m0lit[col] = l0;
      p.m1lit[col] = l1;
    }
    p.outs.push_back({le.e->out, 0, a * d + b, Ty::Double});
  }
  for (int64_t c = 0; c < d; ++c)
    if (p.m0sym[c] == -2) p.m0sym[c] = p.m1sym[c] = -1;   // column not used: any mean
  p.x = X;
  p.keys = Y;
  p.d = d;
  p.nres = d * d;
  p.fam = LoopPlan::GdaScatter;
  p.family = "gda_scatter";
  p.launch = "dlx_gda_pass2";
  return true;
}

// ---- family: logistic regression (collect h = link(theta . x_i) + d residual-weighted sums) -----
// The loop the reference fuses from the collect form: one collect whose value is a
// scalar expression of a nested dot reduce D = sum_j theta(j) * x(i*d + j), and reduces
// g_j = sum_i (h - toDouble(y(i))) * x(i*d + j) reading the collect's value h (vertical fusion).
bool Executor::link_compile(const SEP& f, const SEP& dot, LoopPlan& p, std::unordered_map<const SE*, int>& reg) {
  if (f == dot) return true;   // r[0]
  if (reg.count(f.get())) return true;
  auto emit = [&](uint8_t op, int a, int b, double imm) {
    const int q = p.link.n;
    const int r = static_cast<int>(reg.size()) + 1;
    if (q >= DLX_LINK_MAX_CODE || r >= DLX_LINK_MAX_REGS) return false;
    p.link.op[q] = op;
    p.link.a[q] = static_cast<uint8_t>(a);
    p.link.b[q] = static_cast<uint8_t>(b);
    p.link.imm[q] = imm;
    p.link.dst[q] = static_cast<uint8_t>(r);
    p.link.n = q + 1;
    reg[f.get()] = r;
    return true;
  };
  auto r_of = [&](const SEP& x) { return x == dot ? 0 : reg.at(x.get()); };
  switch (f->k) {
    case SE::Const:
      if (f->ty != Ty::Double) return false;
      return emit(DLX_LINK_CONST, 0, 0, f->cd);
    case SE::Host:
      if (!f->host.is_dbl()) return false;
      p.link_patches.emplace_back(p.link.n, f->sym);
      return emit(DLX_LINK_CONST, 0, 0, f->host.d());
    case SE::Bin: {
      if (f->ty != Ty::Double || !link_compile(f->a[0], dot, p, reg) || !link_compile(f->a[1], dot, p, reg)) return false;
      const uint8_t op = f->op == Op::Plus ? DLX_LINK_ADD : f->op == Op::Minus ? DLX_LINK_SUB
                         : f->op == Op::Times ? DLX_LINK_MUL : f->op == Op::Divide ? DLX_LINK_DIV : 255;
      if (op == 255) return false;
      return emit(op, r_of(f->a[0]), r_of(f->a[1]), 0);
    }
    case SE::Un: {
      if (f->ty != Ty::Double || !link_compile(f->a[0], dot, p, reg)) return false;
      const uint8_t op = f->op == Op::MathAbs ? DLX_LINK_ABS : f->op == Op::MathExp ? DLX_LINK_EXP
                         : f->op == Op::MathSqrt ? DLX_LINK_SQRT : 255;
      if (op == 255) return false;
      return emit(op, r_of(f->a[0]), 0, 0);
    }
    default: return false;
  }
}

bool Executor::match_logistic(const Stmt& s, int64_t n, std::vector<LElem>& els, LoopPlan& p, MatchCtx& m) {
  (void)n;
  int ci = -1;
  for (size_t q = 0; q < els.size(); ++q)
    if (els[q].e->kind == Elem::Collect) {
      if (ci >= 0) MISS("two collects");
      ci = static_cast<int>(q);
    }
  if (ci < 0 || els[ci].cond || els[ci].e->append || els[ci].e->out_ty.elem != Ty::Double) MISS("no dense Double collect");
  const SEP F = els[ci].value;
  // the one nested reduce in F: the dot
  SEP D;
  std::vector<SEP> stack{F};
  while (!stack.empty()) {
    SEP x = stack.back();
    stack.pop_back();
    if (x->k == SE::Red) {
      if (D && D != x) MISS("two nested reduces");
      D = x;
      continue;
    }
    if (x->k == SE::Load || x->k == SE::Idx || x->k == SE::Sel) MISS("link reads beyond the dot");
    for (const SEP& c : x->a) stack.push_back(c);
  }
  if (!D || D->ty != Ty::Double || !is_plus_combine(D->a[1]) || !zero_is_pos0(D->zero)) MISS("no dot reduce");
  const int64_t d = D->range;
  const SEP& prod = D->a[0];
  if (prod->k != SE::Bin || prod->op != Op::Times || prod->a[0]->k != SE::Load || prod->a[1]->k != SE::Load)
    MISS("dot elem is not a product of two loads");
  int xs = -1, ts = -1;
  for (int side = 0; side < 2; ++side) {
    const SEP& ld = prod->a[side];
    Affine af;
    if (!affine(ld->a[1], &af) || ld->a[0]->ty != Ty::Double) MISS("dot load");
    if (af.a == d && af.b == 1 && af.c == 0 && af.inner == D->sym) xs = m.slot(ld->a[0]);
    else if (af.a == 0 && af.b == 1 && af.c == 0 && af.inner == D->sym) ts = m.slot(ld->a[0]);
  }
  if (xs < 0 || ts < 0) MISS("dot is not theta(j) * x(i*d + j)");
  p.link = dlx_link_code{};
  p.link_patches.clear();
  std::unordered_map<const SE*, int> reg;
  if (!link_compile(F, D, p, reg)) MISS("link expression");
  p.link.out = F == D ? 0 : reg.at(F.get());
  // the gradient reduces
  p.outs.clear();
  p.outs.push_back({els[ci].e->out, 1, 0, Ty::Double});
  int ys = -1;
  std::vector<uint8_t> seen(d, 0);
  for (size_t q = 0; q < els.size(); ++q) {
    if (static_cast<int>(q) == ci) continue;
    const LElem& le = els[q];
    if (le.e->kind != Elem::Reduce || le.cond || !is_plus_combine(le.combine) || !zero_is_pos0(le.e->zero))
      MISS("elem is not an unguarded + reduce from 0.0");
    const SEP& v = le.value;
    if (v->k != SE::Bin || v->op != Op::Times) MISS("gradient elem is not a product");
    SEP R = v->a[0], L = v->a[1];
    if (R->k == SE::Load) std::swap(R, L);
    if (L->k != SE::Load || R->k != SE::Bin || R->op != Op::Minus || R->a[0] != F) MISS("not (h - y) * x");
    const SEP& yd = R->a[1];
    if (yd->k != SE::Un || yd->op != Op::ToDouble || yd->a[0]->k != SE::Load || yd->a[0]->a[0]->ty != Ty::Int)
      MISS("label is not toDouble(y(i))");
    Affine ay, ax;
    if (!affine(yd->a[0]->a[1], &ay) || ay.a != 1 || ay.b != 0 || ay.c != 0) MISS("label index is not i");
    const int y = m.slot(yd->a[0]->a[0]);
    if (ys >= 0 && ys != y) MISS("two label vectors");
    ys = y;
    if (!affine(L->a[1], &ax) || m.slot(L->a[0]) != xs || ax.a != d || ax.b != 0 || ax.c < 0 || ax.c >= d)
      MISS("gradient column is not x(i*d + j)");
    if (seen[ax.c]) MISS("column twice");
    seen[ax.c] = 1;
    p.outs.push_back({le.e->out, 0, ax.c, Ty::Double});
  }
  if (ys < 0) MISS("no gradient");
  p.x = xs;
  p.mu = ts;
  p.keys = ys;
  p.d = d;
  p.nres = d;
  // theta(j) = theta(j) - alpha * g_j after the loop (UpdateGroup::Axpy): on the device
  p.upd_vec = -1;
  p.skip.clear();
  p.sums_group_only = false;
  auto g = P.update_after.find(s.sym);
  if (g != P.update_after.end() && g->second.kind == UpdateGroup::Axpy &&
      static_cast<int64_t>(g->second.entries.size()) == d) {
    std::unordered_map<int, int64_t> col;   // gradient out -> column
    for (const LoopPlan::Out& o : p.outs)
      if (o.src == 0) col[o.sym] = o.ix;
    std::vector<uint8_t> cov(d, 0);
    bool ok = true;
    for (const UpdateGroup::Entry& en : g->second.entries) {
      auto c = col.find(en.sum_sym);
      if (c == col.end() || c->second != en.e || cov[en.e]) ok = false;
      else cov[en.e] = 1;
    }
    const Atom& al = g->second.alpha;
    if (ok && (al.k == Atom::Double || al.k == Atom::Sym)) {
      p.upd_vec = g->second.vec_sym;
      p.skip = g->second.stmts;
      p.alpha_sym = al.k == Atom::Sym ? al.sym : -1;
      p.alpha_lit = al.d;
      size_t only = 0;
      for (LoopPlan::Out& o : p.outs) {
        o.group_only = o.src == 0 && P.uses[o.sym] == 1;   // read only by its Times
        only += o.group_only;
      }
      p.sums_group_only = only == static_cast<size_t>(d);
    }
  }
  p.fam = LoopPlan::Logistic;
  p.family = "logistic";
  p.launch = p.upd_vec >= 0 ? "dlx_rowdot_link_grad + dlx_axpy_inplace" : "dlx_rowdot_link_grad";
  return true;
}

// ---- generic multiloop kernel (bytecode) -------------------------------------------------------
int Executor::vm_emit(LoopPlan& p, MatchCtx& m, std::unordered_map<const SE*, int>& reg, int& nreg, const SEP& s) {
  auto it = reg.find(s.get());
  if (it != reg.end()) return it->second;
  auto push = [&](uint8_t op, int a, int b, int64_t imm, int aux) {
    if (nreg >= DLX_VM_MAX_REGS) gen_fail("multiloop body needs more than " + std::to_string(DLX_VM_MAX_REGS) + " registers");
    dlx_vm_instr in{};
    in.op = op;
    in.dst = static_cast<uint8_t>(nreg);
    in.a = static_cast<uint8_t>(a);
    in.b = static_cast<uint8_t>(b);
    in.imm = imm;
    in.aux = aux;
    p.code.push_back(in);
    return nreg++;
  };
  int r = -1;
  switch (s->k) {
    case SE::Const: {
      int64_t bits = s->ci;
      if (s->ty == Ty::Double) std::memcpy(&bits, &s->cd, 8);
      r = push(DLX_VM_CONST, 0, 0, bits, 0);
      break;
    }
    case SE::Host:   // a host scalar: re-read from the environment at every launch
      r = push(DLX_VM_CONST, 0, 0, val_bits(s->host), 0);
      p.patches.emplace_back(static_cast<int>(p.code.size()) - 1, s->sym);
      break;
    case SE::Idx: r = push(DLX_VM_IDX, 0, 0, 0, 0); break;
    case SE::Load: {
      const int vi = m.slot(s->a[0]);
      if (vi >= DLX_VM_MAX_VECS) gen_fail("multiloop reads too many vectors");
      const int ir = vm_emit(p, m, reg, nreg, s->a[1]);
      r = push(DLX_VM_LOAD, ir, 0, 0, vi);
      break;
    }
    case SE::Bin: {
      const int x = vm_emit(p, m, reg, nreg, s->a[0]), y = vm_emit(p, m, reg, nreg, s->a[1]);
      const bool dbl = s->a[0]->ty == Ty::Double;
      uint8_t o;
      switch (s->op) {
        case Op::Plus: o = dbl ? DLX_VM_ADD_D : DLX_VM_ADD_I; break;
        case Op::Minus: o = dbl ? DLX_VM_SUB_D : DLX_VM_SUB_I; break;
        case Op::Times: o = dbl ? DLX_VM_MUL_D : DLX_VM_MUL_I; break;
        case Op::Divide: o = dbl ? DLX_VM_DIV_D : DLX_VM_DIV_I; break;
        case Op::Lt: o = dbl ? DLX_VM_LT_D : DLX_VM_LT_I; break;
        case Op::Eq: o = dbl ? DLX_VM_EQ_D : DLX_VM_EQ_I; break;
        case Op::And: o = DLX_VM_AND; break;
        case Op::Or: o = DLX_VM_OR; break;
        default: gen_fail("binary operator in a multiloop");
      }
      r = push(o, x, y, 0, 0);
      break;
    }
    case SE::Un: {
      const int x = vm_emit(p, m, reg, nreg, s->a[0]);
      uint8_t o;
      switch (s->op) {
        case Op::Not: o = DLX_VM_NOT; break;
        case Op::MathAbs: o = s->ty == Ty::Double ? DLX_VM_ABS_D : DLX_VM_ABS_I; break;
        case Op::MathSqrt: o = DLX_VM_SQRT; break;
        case Op::MathExp: o = DLX_VM_EXP; break;
        case Op::ToDouble: o = DLX_VM_TODBL; break;
        default: gen_fail("unary operator in a multiloop");
      }
      r = push(o, x, 0, 0, 0);
      break;
    }
    case SE::Sel: {
      const int c = vm_emit(p, m, reg, nreg, s->a[0]), t = vm_emit(p, m, reg, nreg, s->a[1]),
                f = vm_emit(p, m, reg, nreg, s->a[2]);
      r = push(DLX_VM_SEL, t, f, c, 0);
      break;
    }
    default: gen_fail("nested reduce in a generic multiloop");
  }
  reg[s.get()] = r;
  return r;
}

static int vm_ty(Ty t) { return t == Ty::Double ? DLX_VM_F64 : t == Ty::Bool ? DLX_VM_BOOL : DLX_VM_I64; }

bool Executor::match_generic(int64_t n, std::vector<LElem>& els, LoopPlan& p, MatchCtx& m) {
  if (els.size() > DLX_VM_MAX_ELEMS) gen_fail("multiloop with more than 16 live elems outside the specialised families");
  p.code.clear();
  p.patches.clear();
  p.outs.clear();
  p.coll_ty.clear();
  dlx_vm_loop& L = p.L;
  L = dlx_vm_loop{};
  L.range = n;
  L.body_end = 0;
  L.nelems = static_cast<int>(els.size());
  for (size_t q = 0; q < els.size(); ++q) {
    const LElem& le = els[q];
    dlx_vm_elem& ve = L.elem[q];
    Ty cty = Ty::Int;
    if (le.e->kind == Elem::Collect) {
      // filter-collect (append): order-preserving compaction, length returned in the result slot
      ve.kind = le.e->append ? DLX_VM_APPEND : DLX_VM_COLLECT;
      cty = le.e->out_ty.elem == Ty::Double ? Ty::Double : le.e->out_ty.elem == Ty::Bool ? Ty::Bool : Ty::Int;
      ve.ty = vm_ty(cty);
      p.outs.push_back({le.e->out, 1, static_cast<int64_t>(q), cty});
    } else if (le.e->kind == Elem::Reduce) {
      ve.kind = DLX_VM_REDUCE;
      ve.ty = vm_ty(le.e->out_ty.t);
      if (is_plus_combine(le.combine)) ve.combine = DLX_VM_COMBINE_ADD;
      else if (is_times_combine(le.combine)) ve.combine = DLX_VM_COMBINE_MUL;
      else gen_fail("reduce combine other than + or *");
      int64_t bits = le.e->zero.i;
      if (le.e->zero.k == Atom::Double) std::memcpy(&bits, &le.e->zero.d, 8);
      if (le.e->zero.k == Atom::Bool) bits = le.e->zero.b;
      if (le.e->zero.k == Atom::Sym) gen_fail("reduce zero that is not a literal");
      ve.zero = bits;
      p.outs.push_back({le.e->out, 0, static_cast<int64_t>(q), le.e->out_ty.t});
    } else {
      gen_fail("foreach elems are not lowered (disjoint-write contract, SPEC.md:673)");
    }
    p.coll_ty.push_back(cty);
    // each elem gets its own code ranges; shared sub-DAGs are re-emitted per elem so a guarded
    // elem never reads a register computed under another elem's guard
    std::unordered_map<const SE*, int> reg;
    int nreg = 0;
    if (le.cond) {
      ve.cond_begin = static_cast<int>(p.code.size());
      ve.cond_reg = vm_emit(p, m, reg, nreg, le.cond);
      ve.cond_end = static_cast<int>(p.code.size());
    } else {
      ve.cond_begin = ve.cond_end = static_cast<int>(p.code.size());
    }
    ve.value_begin = static_cast<int>(p.code.size());
    ve.value_reg = vm_emit(p, m, reg, nreg, le.value);
    ve.value_end = static_cast<int>(p.code.size());
  }
  if (p.code.size() > DLX_VM_MAX_CODE) gen_fail("multiloop body too large for the generic kernel");
  L.ncode = static_cast<int>(p.code.size());
  p.nres = DLX_VM_MAX_ELEMS + 1;
  p.fam = LoopPlan::Generic;
  p.family = "generic";
  p.launch = "dlx_vm_run_loop";
  return true;
}

// ---- lowering, cache, launch -------------------------------------------------------------------
// DLX_PROGRAM_VM=1: loops outside the specialised families run on the bytecode kernel (vm.cu)
// instead of a kernel compiled from the loop body (lower_jit.cpp)
static bool use_vm() {
  static const bool v = getenv("DLX_PROGRAM_VM") && atoi(getenv("DLX_PROGRAM_VM")) != 0;
  return v;
}

std::shared_ptr<LoopPlan> Executor::lower(const Stmt& s, int64_t n) {
  const Loop& L = *s.loop;
  MatchCtx m;
  struct CtxReset {
    Executor* e;
    ~CtxReset() {
      e->mc_ = nullptr;
      e->loop_index_ = -1;
      e->sym_.clear();
    }
  } reset{this};
  mc_ = &m;
  loop_index_ = L.index;
  sym_.clear();
  sym_block(L.body);
  std::vector<LElem> els;
  for (const Elem& e : L.elems) {
    if (!e.live) continue;
    LElem le{&e, nullptr, nullptr, nullptr};
    if (e.cond >= 0) le.cond = sym_block(e.cond);
    le.value = sym_block(e.elem);
    if (e.kind == Elem::Reduce) {
      sym_[e.rv_left] = mk(SE::RvL, e.out_ty.t);
      sym_[e.rv_right] = mk(SE::RvR, e.out_ty.t);
      le.combine = sym_block(e.combine);
    }
    els.push_back(le);
  }
  auto p = std::make_shared<LoopPlan>();
  const bool ok = match_kmeans(s, n, els, *p, m) || match_logistic(s, n, els, *p, m) || match_groupby(n, els, *p, m) ||
                  match_bucket_rows(n, els, *p, m) || match_gda2(n, els, *p, m) ||
                  (use_vm() ? match_generic(n, els, *p, m) : match_compiled(n, els, *p, m));
  if (!ok) gen_fail("multiloop x" + std::to_string(s.sym) + " matches no kernel");
  p->vsyms = m.vsyms;
  for (const VecP& v : m.vecs) {
    p->vtys.push_back(v->elem);
    p->vlens.push_back(v->n);
  }
  p->baked = m.baked;
  p->deps = m.deps;
  return p;
}

// A cached plan applies if the symbols it read are bound, its input vectors have the same
// types and lengths, and every baked host scalar the same value.
bool Executor::plan_valid(const LoopPlan& p, std::vector<VecP>& vecs) {
  for (int dsym : p.deps) {
    if (!bound_[dsym] && !pending_.empty()) join_all();
    if (!bound_[dsym]) return false;
  }
  vecs.clear();
  for (size_t q = 0; q < p.vsyms.size(); ++q) {
    const Val& v = env_[p.vsyms[q]];
    if (!v.is_vec() || v.vec()->elem != p.vtys[q] || v.vec()->n != p.vlens[q]) return false;
    vecs.push_back(v.vec());
  }
  for (const auto& [sym, bits] : p.baked) {
    Val v = force(env_[sym]);
    if ((!v.is_int() && !v.is_dbl() && !v.is_bool()) || val_bits(v) != bits) return false;
  }
  return true;
}

void Executor::bind_empty(const Loop& L) {
  for (const Elem& e : L.elems) {
    if (!e.live) continue;
    if (e.kind == Elem::Collect) {
      const Ty t = e.out_ty.elem == Ty::Double ? Ty::Double : e.out_ty.elem == Ty::Bool ? Ty::Bool : Ty::Int;
      bind(e.out, Val{new_vec(0, t, st_, true)});
    } else if (e.kind == Elem::Reduce) {
      bind(e.out, atomv(e.zero));
    } else {
      bind(e.out, Val{});
    }
  }
}

void Executor::run_loop(const Stmt& s) {
  const Loop& L = *s.loop;
  json rep;
  rep["loop"] = "x" + std::to_string(s.sym);
  const int64_t n = atom(L.range).i();
  if (n <= 0) {   // `while (i < range)` runs no index: every reduce keeps its zero
    bind_empty(L);
    rep["family"] = "empty";
    report.push_back(rep);
    return;
  }
  std::shared_ptr<LoopPlan> plan;
  std::vector<VecP> vecs;
  bool cached = false;
  if (!g_run->dry && !g_run->nocache) {
    std::lock_guard<std::mutex> lk(P.plan_mu);
    auto it = P.plans.find(s.sym);
    if (it != P.plans.end()) plan = it->second;
  }
  if (plan && plan_valid(*plan, vecs)) {
    cached = true;
  } else {
    plan = lower(s, n);
    vecs.clear();
    for (int vs : plan->vsyms) vecs.push_back(env_[vs].vec());
    if (!g_run->dry) {
      std::lock_guard<std::mutex> lk(P.plan_mu);
      P.plans[s.sym] = plan;
    }
  }
  int live = 0;
  for (const Elem& e : L.elems) live += e.live;
  rep["live_elems"] = live;
  rep["family"] = plan->family;
  rep["n"] = n;
  if (plan->fam == LoopPlan::Kmeans) rep["d"] = plan->d, rep["k"] = plan->k;
  if (plan->fam == LoopPlan::GroupBy) rep["buckets"] = plan->k;
  if (plan->fam == LoopPlan::BucketRows) rep["buckets"] = plan->k, rep["d"] = plan->d;
  if (plan->fam == LoopPlan::GdaScatter || plan->fam == LoopPlan::Logistic) rep["d"] = plan->d;
  if (plan->fam == LoopPlan::Logistic) {
    const int lk = dlx_link_kind(&plan->link);
    rep["link"] = lk == 1 ? "sigmoid" : lk == 2 ? "softsign" : "code";
  }
  if (plan->fam == LoopPlan::Generic) rep["elems"] = live, rep["instructions"] = static_cast<int>(plan->code.size());
  if (plan->fam == LoopPlan::Compiled) {
    rep["elems"] = live;
    rep["source_bytes"] = static_cast<int64_t>(plan->jit_src.size());
  }
  rep["launch"] = plan->launch;
  rep["cached"] = cached;
  if (g_run->dry) {
    dry_n_ = n;
    for (const LoopPlan::Out& o : plan->outs) {
      if (o.src == 1) bind(o.sym, Val{new_vec(dry_n_, o.ty, st_, false)});
      else if (o.ty == Ty::Double) bind(o.sym, Val{1.0});
      else if (o.ty == Ty::Bool) bind(o.sym, Val{false});
      else bind(o.sym, Val{int64_t{1}});
    }
    if (plan->upd_vec >= 0) rep["update"] = "device";
    report.push_back(rep);
    return;
  }
  flush_mirrors();
  // next loop stream, ordered after everything the main stream has enqueued so far (RNG fills,
  // uploads, mirror flushes: the loop's inputs)
  static const int nstreams = getenv("DLX_PROGRAM_STREAMS") ? std::max(1, std::min(kLoopStreams, atoi(getenv("DLX_PROGRAM_STREAMS")))) : kLoopStreams;
  lst_ = res_->loop[launches_++ % nstreams];
  cudaEvent_t ev = get_event();
  ckc(cudaEventRecord(ev, st_), "cudaEventRecord");
  ckc(cudaStreamWaitEvent(lst_, ev, 0), "cudaStreamWaitEvent");
  res_->events.push_back(ev);
  const size_t inflight = pending_.size();
  const auto t0 = std::chrono::steady_clock::now();
  cudaEvent_t pe0 = nullptr, pe1 = nullptr;
  if (g_run->profile) {   // device time of the loop's launches (from its stream's start)
    cudaEventCreate(&pe0);
    cudaEventCreate(&pe1);
    cudaEventRecord(pe0, lst_);
  }
  launch(s, *plan, n, vecs, rep);
  if (g_run->profile) {
    cudaEventRecord(pe1, lst_);
    fprintf(stderr, "[dlx profile] @%.2f ms x%d launch %.1f us (in flight %zu)\n", g_run->ms(), s.sym,
            std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count(), inflight);
    pending_.push_back(Pending{get_event(), [pe0, pe1, sym = s.sym, t0ev = prof_t0_] {
                                 float ms = 0, a = 0, b = 0;
                                 cudaEventElapsedTime(&ms, pe0, pe1);
                                 cudaEventElapsedTime(&a, t0ev, pe0);
                                 cudaEventElapsedTime(&b, t0ev, pe1);
                                 fprintf(stderr, "[dlx profile] x%d device %.1f us [%.1f, %.1f] us from run start\n", sym,
                                         ms * 1e3, a * 1e3, b * 1e3);
                                 cudaEventDestroy(pe0);
                                 cudaEventDestroy(pe1);
                               }});
    cudaEventRecord(pending_.back().ev, lst_);
  }
  rep["stream"] = static_cast<int>((launches_ - 1) % kLoopStreams);
  rep["in_flight"] = static_cast<int>(inflight);   // loops it may overlap
  report.push_back(rep);
  if (g_run->serial) join_all();
}

void Executor::launch(const Stmt& s, LoopPlan& p, int64_t n, std::vector<VecP>& vecs, json& rep) {
  if (sharded(p)) {   // contiguous index shards over ExecOptions.devices (shard.cpp)
    rep["shards"] = static_cast<int>(devs_.size());
    switch (p.fam) {
      case LoopPlan::Kmeans: launch_kmeans_sharded(p, n, vecs, rep); return;
      case LoopPlan::GroupBy: launch_groupby_sharded(p, n, vecs); return;
      case LoopPlan::BucketRows: launch_bucket_rows_sharded(p, n, vecs); return;
      case LoopPlan::GdaScatter: launch_gda2_sharded(p, n, vecs); return;
      case LoopPlan::Logistic: launch_logistic_sharded(p, n, vecs, rep); return;
      default: break;
    }
  }
  switch (p.fam) {
    case LoopPlan::Kmeans: launch_kmeans(s, p, n, vecs, rep); break;
    case LoopPlan::GroupBy: launch_groupby(p, n, vecs); break;
    case LoopPlan::BucketRows: launch_bucket_rows(p, n, vecs); break;
    case LoopPlan::GdaScatter: launch_gda2(p, n, vecs); break;
    case LoopPlan::Logistic: launch_logistic(p, n, vecs, rep); break;
    case LoopPlan::Generic: launch_generic(p, n, vecs); break;
    case LoopPlan::Compiled: launch_compiled(p, n, vecs); break;
  }
}

void* Executor::dalloc(size_t bytes) {
  void* p = nullptr;
  ckc(cudaMallocAsync(&p, std::max<size_t>(bytes, 16), lst_), "cudaMallocAsync");
  return p;
}
void Executor::dfree(void* p) {
  if (p) cudaFreeAsync(p, lst_);
}

// the loop stream waits for pending device writes of its inputs (DEG data edges); int32-stored
// Int vectors become int64 for the kernels
void Executor::wait_inputs(const std::vector<VecP>& V) {
  for (const VecP& v : V) {
    if (v->wev) cudaStreamWaitEvent(lst_, v->wev, 0);
    if (v->i32) widen(v, lst_);
  }
}

void Executor::bind_scalars(const LoopPlan& p, const int64_t* hres) {
  for (const LoopPlan::Out& o : p.outs)
    if (o.src == 0) bind(o.sym, Val{make_lazy(hres + o.ix, o.ty, 8)});
}

[[noreturn]] static void load_trap() { trap("TrapIndexOutOfBounds: element load out of range in a multiloop"); }

void Executor::launch_kmeans(const Stmt& s, LoopPlan& p, int64_t n, std::vector<VecP>& V, json& rep) {
  (void)s;
  const VecP& x = V[p.x];
  const VecP& mu = V[p.mu];
  const int d = static_cast<int>(p.d), k = static_cast<int>(p.k);
  if (n * d > x->n || static_cast<int64_t>(k) * d > mu->n) load_trap();
  wait_inputs(V);
  VecP U;   // the update group's target, when it can run on the device
  if (p.upd_vec >= 0 && bound_[p.upd_vec] && env_[p.upd_vec].is_vec()) {
    U = env_[p.upd_vec].vec();
    if (U->elem != Ty::Double || U->n != static_cast<int64_t>(k) * d || U->i32) U = nullptr;
  }
  if (U) {
    fence_on(lst_);   // WAR: loops in flight may still read U
    if (U->wev) cudaStreamWaitEvent(lst_, U->wev, 0);
  }
  const bool copy_sums = !U || !p.sums_group_only;
  const size_t wsb = dlx_kmeans_workspace_bytes(n, d, k);
  void* ws = dalloc(wsb);
  VecP assign = new_vec(n, Ty::Int, lst_, false, /*i32=*/true);
  auto* counts = static_cast<int64_t*>(dalloc(static_cast<size_t>(k) * 8));
  auto* sums = static_cast<double*>(dalloc(static_cast<size_t>(k) * d * 8));
  int rc;
  if (U && U == mu) {
    rc = dlx_kmeans_iteration(static_cast<const double*>(x->p), n, d, k, static_cast<double*>(mu->p),
                              static_cast<int32_t*>(assign->p), counts, sums, ws, wsb, DLX_KMEANS_AUTO, lst_);
  } else {
    rc = dlx_kmeans_step(static_cast<const double*>(x->p), n, d, k, static_cast<const double*>(mu->p),
                         static_cast<int32_t*>(assign->p), counts, sums, ws, wsb, DLX_KMEANS_AUTO, lst_);
    if (rc == DLX_OK && U) rc = dlx_kmeans_update(counts, sums, k, d, static_cast<double*>(U->p), lst_);
  }
  int64_t* hres = res_->pin.get_n<int64_t>(p.nres);
  if (rc == DLX_OK) {
    cudaMemcpyAsync(hres, counts, static_cast<size_t>(k) * 8, cudaMemcpyDeviceToHost, lst_);
    if (copy_sums) cudaMemcpyAsync(hres + k, sums, static_cast<size_t>(k) * d * 8, cudaMemcpyDeviceToHost, lst_);
  }
  dfree(ws);
  dfree(counts);
  dfree(sums);
  ck(rc);
  cudaEvent_t ev = complete_loop({}, nullptr);
  assign->wev = ev;
  for (const LoopPlan::Out& o : p.outs) {
    if (o.src == 1) bind(o.sym, Val{assign});
    else if (!(U && o.group_only)) bind(o.sym, Val{make_lazy(hres + o.ix, o.ty, 8)});
  }
  if (U) {   // the group's k*d host statements ran on the device
    U->wev = ev;
    U->host_valid = false;
    U->page_valid = false;
    U->touched();
    for (int q : p.skip) mark_skip(q);
  }
  rep["update"] = U ? "device" : p.upd_vec >= 0 ? "host" : "none";
}

void Executor::launch_groupby(LoopPlan& p, int64_t n, std::vector<VecP>& V) {
  const VecP& keys = V[p.keys];
  if (n > keys->n) load_trap();
  wait_inputs(V);
  const int64_t nb = p.k;
  const size_t wsb = dlx_groupby_workspace_bytes(n, nb);
  void* ws = dalloc(wsb);
  auto* counts = static_cast<int64_t*>(dalloc(nb * 8));
  int rc = dlx_groupby_count(static_cast<const int64_t*>(keys->p), n, nb, counts, ws, wsb, lst_);
  int64_t* hres = res_->pin.get_n<int64_t>(nb);
  if (rc == DLX_OK) cudaMemcpyAsync(hres, counts, nb * 8, cudaMemcpyDeviceToHost, lst_);
  dfree(ws);
  dfree(counts);
  ck(rc);
  complete_loop({}, nullptr);
  bind_scalars(p, hres);
}

void Executor::launch_bucket_rows(LoopPlan& p, int64_t n, std::vector<VecP>& V) {
  const VecP& x = V[p.x];
  const VecP& keys = V[p.keys];
  if (n > keys->n || n * p.d > x->n) load_trap();
  wait_inputs(V);
  const int32_t d = static_cast<int32_t>(p.d), K = static_cast<int32_t>(p.k);
  const size_t wsb = dlx_bucket_rowsum_workspace_bytes(n, d, K);
  void* ws = dalloc(wsb);
  auto* rec = static_cast<int64_t*>(dalloc(p.nres * 8));   // counts[K], then sums[K][d]
  int rc = dlx_bucket_rowsum(static_cast<const double*>(x->p), static_cast<const int64_t*>(keys->p), n, d,
                             p.buckets.data(), K, rec, reinterpret_cast<double*>(rec + K), ws, wsb, lst_);
  int64_t* hres = res_->pin.get_n<int64_t>(p.nres);
  if (rc == DLX_OK) cudaMemcpyAsync(hres, rec, p.nres * 8, cudaMemcpyDeviceToHost, lst_);
  dfree(ws);
  dfree(rec);
  ck(rc);
  complete_loop({}, nullptr);
  bind_scalars(p, hres);
}

void Executor::launch_gda2(LoopPlan& p, int64_t n, std::vector<VecP>& V) {
  const VecP& X = V[p.x];
  const VecP& Y = V[p.keys];
  const int64_t d = p.d;
  if (n * d > X->n || n > Y->n) load_trap();
  // the class means: host scalars of this run (or literals)
  double* hmu = res_->pin.get_n<double>(2 * d);
  for (int64_t c = 0; c < d; ++c) {
    hmu[c] = p.m0sym[c] >= 0 ? force(env_[p.m0sym[c]]).d() : p.m0lit[c];
    hmu[d + c] = p.m1sym[c] >= 0 ? force(env_[p.m1sym[c]]).d() : p.m1lit[c];
  }
  wait_inputs(V);
  const size_t wsb = dlx_gda_workspace_bytes(n, static_cast<int32_t>(d));
  auto* dmu = static_cast<double*>(dalloc(2 * d * 8));
  auto* S = static_cast<double*>(dalloc(d * d * 8));
  void* ws = dalloc(wsb);
  cudaMemcpyAsync(dmu, hmu, 2 * d * 8, cudaMemcpyHostToDevice, lst_);
  int rc = dlx_gda_pass2(static_cast<const double*>(X->p), static_cast<const int64_t*>(Y->p), n, static_cast<int32_t>(d),
                         dmu, dmu + d, S, ws, wsb, lst_);
  int64_t* hres = res_->pin.get_n<int64_t>(d * d);
  if (rc == DLX_OK) cudaMemcpyAsync(hres, S, d * d * 8, cudaMemcpyDeviceToHost, lst_);
  dfree(dmu);
  dfree(S);
  dfree(ws);
  ck(rc);
  complete_loop({}, nullptr);
  bind_scalars(p, hres);
}

void Executor::launch_logistic(LoopPlan& p, int64_t n, std::vector<VecP>& V, json& rep) {
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
    fence_on(lst_);   // WAR: loops in flight may still read U
    if (U->wev) cudaStreamWaitEvent(lst_, U->wev, 0);
  }
  const bool copy_grad = !U || !p.sums_group_only;
  VecP h = new_vec(n, Ty::Double, lst_, false);
  const size_t wsb = dlx_logreg_workspace_bytes(n, d);
  void* ws = dalloc(wsb);
  auto* grad = static_cast<double*>(dalloc(static_cast<size_t>(d) * 8));
  int rc = dlx_rowdot_link_grad(static_cast<const double*>(X->p), static_cast<const int64_t*>(Y->p), n, d,
                                static_cast<const double*>(TH->p), &link, static_cast<double*>(h->p), grad, ws, wsb, lst_);
  if (rc == DLX_OK && U) rc = dlx_axpy_inplace(static_cast<double*>(U->p), grad, alpha, d, lst_);
  int64_t* hres = res_->pin.get_n<int64_t>(d);
  if (rc == DLX_OK && copy_grad) cudaMemcpyAsync(hres, grad, static_cast<size_t>(d) * 8, cudaMemcpyDeviceToHost, lst_);
  dfree(ws);
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

void Executor::launch_generic(LoopPlan& p, int64_t n, std::vector<VecP>& V) {
  wait_inputs(V);
  dlx_vm_loop L = p.L;
  L.range = n;
  L.nvecs = static_cast<int>(V.size());
  if (L.nvecs > DLX_VM_MAX_VECS) gen_fail("multiloop reads too many vectors");
  for (size_t q = 0; q < V.size(); ++q) {
    L.vec[q] = V[q]->p;
    L.vec_len[q] = V[q]->n;
    L.vec_kind[q] = vm_ty(V[q]->elem);
  }
  std::vector<VecP> outs(L.nelems);
  for (int q = 0; q < L.nelems; ++q)
    if (L.elem[q].kind != DLX_VM_REDUCE) {
      outs[q] = new_vec(n, p.coll_ty[q], lst_, true);
      L.elem[q].out = outs[q]->p;
    }
  const size_t wsb = dlx_vm_workspace_bytes(n);
  const size_t code_bytes = std::max<size_t>(1, p.code.size()) * sizeof(dlx_vm_instr);
  auto* dcode = static_cast<dlx_vm_instr*>(dalloc(code_bytes));
  auto* dres = static_cast<int64_t*>(dalloc((DLX_VM_MAX_ELEMS + 1) * 8));   // results, then the trap word
  auto* dtrap = reinterpret_cast<uint64_t*>(dres + DLX_VM_MAX_ELEMS);
  void* ws = dalloc(wsb);
  // staged through pinned memory so the copies (and the launch) do not block the host
  auto* hcode = res_->pin.get_n<dlx_vm_instr>(std::max<size_t>(1, p.code.size()));
  if (!p.code.empty()) std::memcpy(hcode, p.code.data(), p.code.size() * sizeof(dlx_vm_instr));
  for (auto [ix, sym] : p.patches) hcode[ix].imm = val_bits(force(env_[sym]));
  auto* zeros = res_->pin.get_n<int64_t>(DLX_VM_MAX_ELEMS + 1);
  std::memset(zeros, 0, (DLX_VM_MAX_ELEMS + 1) * 8);
  for (int q = 0; q < L.nelems; ++q) zeros[q] = L.elem[q].zero;
  zeros[DLX_VM_MAX_ELEMS] = -1;   // the trap word: UINT64_MAX = no trap
  cudaMemcpyAsync(dcode, hcode, p.code.size() * sizeof(dlx_vm_instr), cudaMemcpyHostToDevice, lst_);
  cudaMemcpyAsync(dres, zeros, (DLX_VM_MAX_ELEMS + 1) * 8, cudaMemcpyHostToDevice, lst_);
  int rc = dlx_vm_run_loop(dcode, &L, dres, dtrap, ws, wsb, lst_);
  int64_t* res = res_->pin.get_n<int64_t>(DLX_VM_MAX_ELEMS + 1);
  if (rc == DLX_OK) cudaMemcpyAsync(res, dres, (DLX_VM_MAX_ELEMS + 1) * 8, cudaMemcpyDeviceToHost, lst_);
  dfree(dcode);
  dfree(dres);
  dfree(ws);
  ck(rc);
  std::vector<int> out_syms;
  for (const LoopPlan::Out& o : p.outs) out_syms.push_back(o.sym);
  const std::vector<LoopPlan::Out> po = p.outs;
  std::vector<uint8_t> append(L.nelems);
  for (int q = 0; q < L.nelems; ++q) append[q] = L.elem[q].kind == DLX_VM_APPEND;
  // deferred binding: traps and appended lengths are known only when the loop completes
  complete_loop(out_syms, [this, res, po, outs, append] {
    uint64_t htrap;
    std::memcpy(&htrap, res + DLX_VM_MAX_ELEMS, sizeof(htrap));
    if (htrap != ~0ull) {   // the first trap in index order, as sequential execution meets it
      const std::string at = " at index " + std::to_string(htrap >> 2);
      switch (static_cast<int>(htrap & 3)) {
        case DLX_VM_TRAP_DIV0: trap("TrapDivByZero: integer division by zero in a multiloop" + at);
        case DLX_VM_TRAP_BOUNDS: trap("TrapIndexOutOfBounds: element load out of range in a multiloop" + at);
        default: gen_fail("generic kernel met an unknown instruction");
      }
    }
    for (const LoopPlan::Out& o : po) {
      if (o.src == 1) {
        const VecP& v = outs[o.ix];
        if (append[o.ix]) v->n = res[o.ix];   // the builder's final length
        bind(o.sym, Val{v});
      } else {
        bind(o.sym, lazy_val(Lazy{nullptr, res[o.ix], o.ty, 8, true}));
      }
    }
  });
}

}  // namespace dlx
