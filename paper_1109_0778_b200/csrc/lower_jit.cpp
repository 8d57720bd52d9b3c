// lower_jit.cpp — the generic lowering: a root multiloop that none of the specialised families
// (lower.cpp) matches is rendered as CUDA C++ — ONE kernel whose per-index body is the loop's
// elems, straight-line, in the order emit_parallel_loop renders them (codegen.cpp:345-433) —
// compiled at run time for sm_100a by NVRTC (jit.cpp) and launched on the loop's stream.
//
// What the generated kernel does for index i (the reference's `while (i < range)` body):
//   for each live elem, in order: cond (if any); if it holds, the value; then
//     Collect  out[i] = value                      (loops.cpp:10-103)
//     Append   ordered stream compaction (a count pass + an exclusive scan over CTAs give each
//              CTA its output offset; the main pass compacts in index order; loops.cpp:105-109)
//     Reduce   acc = combine(acc, value)           (+ or *; the elem's zero is folded once, by
//              the final kernel, before the CTA partials in ascending order: codegen.cpp:367-369)
// Nested reduces (an inner multiloop over a loop-invariant range, e.g. a distance or a dot
// product) become sequential inner `for` loops folding left from their zero — exactly the
// reference's inner `while` — so no elem-count, register or nesting cap applies.
// IfThenElse evaluates only the taken branch (MiniC's `if`), Int arithmetic wraps, Int
// division by zero and out-of-range element loads trap: the first trap in index order is
// recorded (atomicMin of index << 2 | kind) and the index is abandoned.  fp64 arithmetic uses
// the round-to-nearest intrinsics and NVRTC runs with --fmad=false: no contraction, so every
// elem value is bit-identical to the sequential reference; only the reduce order differs (the
// chunked executeDEG's ascending combine).
#include <cinttypes>
#include <cstring>
#include <unordered_map>

#include "jit.hpp"
#include "program_exec.hpp"

namespace dlx {
void count_launch();
}

namespace dlx {

namespace {

const char* kPrelude = R"(typedef long long i64;
typedef unsigned long long u64;
__device__ __forceinline__ double dbits(u64 b) { return __longlong_as_double((i64)b); }
__device__ __forceinline__ u64 bitsd(double d) { return (u64)__double_as_longlong(d); }
__device__ __forceinline__ i64 iadd(i64 a, i64 b) { return (i64)((u64)a + (u64)b); }
__device__ __forceinline__ i64 isub(i64 a, i64 b) { return (i64)((u64)a - (u64)b); }
__device__ __forceinline__ i64 imul(i64 a, i64 b) { return (i64)((u64)a * (u64)b); }
__device__ __forceinline__ i64 idiv(i64 a, i64 b) { return (a == (i64)0x8000000000000000ULL && b == -1) ? a : a / b; }
__device__ __forceinline__ i64 iabs(i64 a) { return a < 0 ? (i64)(0ULL - (u64)a) : a; }
__device__ __forceinline__ double cadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ i64 cadd(i64 a, i64 b) { return iadd(a, b); }
__device__ __forceinline__ double cmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ i64 cmul(i64 a, i64 b) { return imul(a, b); }
__device__ __forceinline__ double shfl(double v, int o) { return __shfl_xor_sync(0xffffffffu, v, o); }
__device__ __forceinline__ i64 shfl(i64 v, int o) { return __shfl_xor_sync(0xffffffffu, v, o); }
__device__ __forceinline__ void trap_at(u64* t, i64 i, int kind) { atomicMin(t, ((u64)i << 2) | (u64)kind); }
__device__ __forceinline__ u64 tobits(double v) { return bitsd(v); }
__device__ __forceinline__ u64 tobits(i64 v) { return (u64)v; }
__device__ __forceinline__ void frombits(u64 b, double& v) { v = dbits(b); }
__device__ __forceinline__ void frombits(u64 b, i64& v) { v = (i64)b; }
)";

// W (u64 words, device memory) layout
enum : int { kWRange = 0, kWChunk, kWParts, kWCounts, kWOffsets, kWRes, kWTrap, kWHead };
constexpr int kJitThreads = 256;
constexpr int kJitMaxElems = 1024;
constexpr int kFoldChunk = 64;   // reduce elems folded per shared-memory round

std::string ctype(Ty t) {
  switch (t) {
    case Ty::Int: return "i64";
    case Ty::Double: return "double";
    case Ty::Bool: return "bool";
    default: gen_fail("multiloop value of a non-scalar type");
  }
}

int64_t val_bits_of(const Val& v) {
  if (v.is_int()) return v.i();
  if (v.is_bool()) return v.b();
  if (v.is_dbl()) {
    int64_t b;
    const double d = v.d();
    std::memcpy(&b, &d, 8);
    return b;
  }
  gen_fail("multiloop reads a host value that is not a scalar");
}

bool is_rv_pair(const SEP& c, Op op) {
  return c && c->k == SE::Bin && c->op == op &&
         ((c->a[0]->k == SE::RvL && c->a[1]->k == SE::RvR) || (c->a[0]->k == SE::RvR && c->a[1]->k == SE::RvL));
}
bool is_plus_combine(const SEP& c) { return is_rv_pair(c, Op::Plus); }
bool is_times_combine(const SEP& c) { return is_rv_pair(c, Op::Times); }

std::string hex64(uint64_t b) {
  char buf[32];
  snprintf(buf, sizeof buf, "0x%016" PRIx64 "ULL", b);
  return buf;
}

struct CGen {
  // inputs
  MatchCtx& m;
  std::vector<int>& host_syms;   // W slot -> env symbol
  int nv_max = 64;
  // output
  std::string out;
  int ind = 1;
  int nvar = 0;
  std::string trap_label;
  std::vector<std::unordered_map<const SE*, std::string>> scopes{1};
  std::unordered_map<int, std::string> inner;   // inner index symbol -> C variable
  std::string rv_l, rv_r;                        // the accumulator / value inside a combine
  std::unordered_map<int, int> host_slot;

  CGen(MatchCtx& mc, std::vector<int>& hs) : m(mc), host_syms(hs) {}

  void line(const std::string& s) {
    out.append(2 * ind, ' ');
    out += s;
    out += '\n';
  }
  std::string fresh() { return "v" + std::to_string(nvar++); }
  const std::string* find(const SE* s) const {
    for (auto it = scopes.rbegin(); it != scopes.rend(); ++it) {
      auto f = it->find(s);
      if (f != it->end()) return &f->second;
    }
    return nullptr;
  }
  void open() {
    ++ind;
    scopes.emplace_back();
  }
  void close() {
    scopes.pop_back();
    --ind;
  }
  std::string def(const SEP& s, const std::string& expr) {
    const std::string v = fresh();
    line("const " + ctype(s->ty) + " " + v + " = " + expr + ";");
    scopes.back()[s.get()] = v;
    return v;
  }
  std::string vec_ref(int q, const char* what) { return std::string(what) + std::to_string(q); }

  std::string gen(const SEP& s) {
    if (const std::string* v = find(s.get())) return *v;
    switch (s->k) {
      case SE::Const:
        if (s->ty == Ty::Double) {
          uint64_t b;
          std::memcpy(&b, &s->cd, 8);
          return "dbits(" + hex64(b) + ")";
        }
        if (s->ty == Ty::Bool) return s->ci ? "true" : "false";
        if (s->ty == Ty::Int) return "((i64)" + hex64(static_cast<uint64_t>(s->ci)) + ")";
        gen_fail("Unit value used inside a multiloop");
      case SE::Idx: return "i";
      case SE::Inner: {
        auto it = inner.find(s->sym);
        if (it == inner.end()) gen_fail("inner index used outside its loop");
        return it->second;
      }
      case SE::Host: {
        auto it = host_slot.find(s->sym);
        int slot;
        if (it == host_slot.end()) {
          slot = static_cast<int>(host_syms.size());
          host_syms.push_back(s->sym);
          host_slot[s->sym] = slot;
        } else {
          slot = it->second;
        }
        const std::string w = "H" + std::to_string(slot);
        if (s->ty == Ty::Double) return "dbits(" + w + ")";
        if (s->ty == Ty::Bool) return "(" + w + " != 0ULL)";
        return "((i64)" + w + ")";
      }
      case SE::Load: {
        const int q = m.slot(s->a[0]);
        if (q >= nv_max) gen_fail("multiloop reads more than " + std::to_string(nv_max) + " vectors");
        const std::string ix = gen(s->a[1]);
        const std::string iv = fresh();
        line("const i64 " + iv + " = " + ix + ";");
        line("if ((u64)" + iv + " >= (u64)N" + std::to_string(q) + ") { trap_at(trap, i, 2); goto " + trap_label + "; }");
        const Ty et = s->a[0]->ty;   // the vector's element type
        std::string e = "V" + std::to_string(q) + "[" + iv + "]";
        if (et == Ty::Bool) e = "(" + e + " != 0)";
        return def(s, e);
      }
      case SE::Bin: {
        const std::string a = gen(s->a[0]), b = gen(s->a[1]);
        const bool dbl = s->a[0]->ty == Ty::Double;
        switch (s->op) {
          case Op::Plus: return def(s, dbl ? "__dadd_rn(" + a + ", " + b + ")" : "iadd(" + a + ", " + b + ")");
          case Op::Minus: return def(s, dbl ? "__dsub_rn(" + a + ", " + b + ")" : "isub(" + a + ", " + b + ")");
          case Op::Times: return def(s, dbl ? "__dmul_rn(" + a + ", " + b + ")" : "imul(" + a + ", " + b + ")");
          case Op::Divide:
            if (dbl) return def(s, "__ddiv_rn(" + a + ", " + b + ")");
            line("if (" + b + " == 0) { trap_at(trap, i, 1); goto " + trap_label + "; }");
            return def(s, "idiv(" + a + ", " + b + ")");
          case Op::Lt: return def(s, "(" + a + " < " + b + ")");
          case Op::Eq: return def(s, "(" + a + " == " + b + ")");
          case Op::And: return def(s, "(" + a + " && " + b + ")");
          case Op::Or: return def(s, "(" + a + " || " + b + ")");
          default: gen_fail("binary operator in a multiloop");
        }
      }
      case SE::Un: {
        const std::string a = gen(s->a[0]);
        switch (s->op) {
          case Op::Not: return def(s, "(!" + a + ")");
          case Op::MathAbs: return def(s, s->ty == Ty::Double ? "fabs(" + a + ")" : "iabs(" + a + ")");
          case Op::MathSqrt: return def(s, "__dsqrt_rn(" + a + ")");
          case Op::MathExp: return def(s, "exp(" + a + ")");
          case Op::ToDouble: return def(s, "__ll2double_rn(" + a + ")");
          default: gen_fail("unary operator in a multiloop");
        }
      }
      case SE::Sel: {
        // only the taken branch runs (MiniC `if`), so a guarded load cannot trap spuriously
        const std::string c = gen(s->a[0]);
        const std::string v = fresh();
        line(ctype(s->ty) + " " + v + ";");
        line("if (" + c + ") {");
        open();
        line(v + " = " + gen(s->a[1]) + ";");
        close();
        line("} else {");
        open();
        line(v + " = " + gen(s->a[2]) + ";");
        close();
        line("}");
        scopes.back()[s.get()] = v;
        return v;
      }
      case SE::Red: {
        // nested reduce: the reference's inner `var acc = zero; while (j < range) acc = comb(acc, e)`
        const std::string r = fresh(), j = fresh();
        std::string z;
        if (s->zero.k == Atom::Int) z = "((i64)" + hex64(static_cast<uint64_t>(s->zero.i)) + ")";
        else if (s->zero.k == Atom::Double) {
          uint64_t b;
          std::memcpy(&b, &s->zero.d, 8);
          z = "dbits(" + hex64(b) + ")";
        } else if (s->zero.k == Atom::Bool) z = s->zero.b ? "true" : "false";
        else gen_fail("nested reduce zero that is not a literal");
        line(ctype(s->ty) + " " + r + " = " + z + ";");
        line("for (i64 " + j + " = 0; " + j + " < " + std::to_string(s->range) + "LL; ++" + j + ") {");
        open();
        const auto saved = inner.find(s->sym) != inner.end() ? inner[s->sym] : std::string();
        inner[s->sym] = j;
        const std::string e = gen(s->a[0]);
        const std::string sl = rv_l, sr = rv_r;
        rv_l = r;
        rv_r = e;
        open();   // the combine's nodes read the accumulator: never reuse them across iterations
        const std::string c = gen(s->a[1]);
        line(r + " = " + c + ";");
        close();
        rv_l = sl;
        rv_r = sr;
        if (saved.empty()) inner.erase(s->sym);
        else inner[s->sym] = saved;
        close();
        line("}");
        scopes.back()[s.get()] = r;
        return r;
      }
      case SE::RvL:
        if (rv_l.empty()) gen_fail("reduce combine operand outside a combine");
        return rv_l;
      case SE::RvR:
        if (rv_r.empty()) gen_fail("reduce combine operand outside a combine");
        return rv_r;
      case SE::Vec: gen_fail("a whole vector used as a value inside a multiloop");
    }
    gen_fail("unknown expression in a multiloop");
  }
};

}  // namespace

bool Executor::match_compiled(int64_t n, std::vector<LElem>& els, LoopPlan& p, MatchCtx& m) {
  const int ne = static_cast<int>(els.size());
  if (ne > kJitMaxElems) gen_fail("multiloop with more than " + std::to_string(kJitMaxElems) + " live elems outside the specialised families");
  p.outs.clear();
  p.coll_ty.clear();
  p.jit_kind.assign(ne, 0);
  p.jit_host.clear();
  std::vector<int> red_of(ne, -1), app_of(ne, -1);
  std::vector<Ty> ety(ne);
  std::vector<int> comb(ne, 0);   // 0 add, 1 mul
  int nred = 0, napp = 0;
  for (int q = 0; q < ne; ++q) {
    const LElem& le = els[q];
    Ty cty = Ty::Int;
    if (le.e->kind == Elem::Collect) {
      cty = le.e->out_ty.elem == Ty::Double ? Ty::Double : le.e->out_ty.elem == Ty::Bool ? Ty::Bool : Ty::Int;
      p.jit_kind[q] = le.e->append ? 2 : 1;
      if (le.e->append) app_of[q] = napp++;
      ety[q] = cty;
      p.outs.push_back({le.e->out, 1, static_cast<int64_t>(q), cty});
    } else if (le.e->kind == Elem::Reduce) {
      ety[q] = le.e->out_ty.t;
      if (ety[q] != Ty::Int && ety[q] != Ty::Double) gen_fail("reduce of a non-numeric type");
      if (is_plus_combine(le.combine)) comb[q] = 0;
      else if (is_times_combine(le.combine)) comb[q] = 1;
      else gen_fail("reduce combine other than + or * (the CTA tree needs an associative combine)");
      if (le.e->zero.k != Atom::Int && le.e->zero.k != Atom::Double) gen_fail("reduce zero that is not a numeric literal");
      red_of[q] = nred++;
      p.outs.push_back({le.e->out, 0, static_cast<int64_t>(q), ety[q]});
    } else {
      gen_fail("foreach elems are not lowered (disjoint-write contract, SPEC.md:673)");
    }
    p.coll_ty.push_back(cty);
  }
  p.jit_nred = nred;
  p.jit_napp = napp;

  // ---- per-index bodies ------------------------------------------------------------------
  // main pass: every elem; count pass: only the append elems' conds
  auto body = [&](bool count_pass, const std::string& label) {
    CGen g(m, p.jit_host);
    g.trap_label = label;
    g.ind = 3;
    for (int q = 0; q < ne; ++q) {
      const LElem& le = els[q];
      const int kind = p.jit_kind[q];
      if (count_pass && kind != 2) continue;
      std::string c;
      if (le.cond) c = g.gen(le.cond);
      if (count_pass) {
        g.line("cnt" + std::to_string(app_of[q]) + " += " + (le.cond ? "(" + c + " ? 1 : 0)" : std::string("1")) + ";");
        continue;
      }
      if (le.cond) {
        g.line("if (" + c + ") {");
        g.open();
      }
      const std::string v = g.gen(le.value);
      const std::string qs = std::to_string(q);
      if (kind == 0) {
        const std::string a = "acc" + std::to_string(red_of[q]);
        g.line(a + " = " + (comb[q] ? "cmul(" : "cadd(") + a + ", " + v + ");");
      } else if (kind == 1) {
        if (ety[q] == Ty::Bool) g.line("((unsigned char*)O" + qs + ")[i] = (unsigned char)(" + v + " ? 1 : 0);");
        else g.line("((" + ctype(ety[q]) + "*)O" + qs + ")[i] = " + v + ";");
      } else {
        const std::string a = std::to_string(app_of[q]);
        g.line("tk" + a + " = true;");
        g.line("av" + a + " = " + v + ";");
      }
      if (le.cond) {
        g.close();
        g.line("}");
      }
    }
    return g.out;
  };
  const std::string main_body = body(false, "L_trap");
  const std::string count_body = napp ? body(true, "L_trap") : std::string();
  const int nv = static_cast<int>(m.vsyms.size());
  const int nh = static_cast<int>(p.jit_host.size());

  // ---- kernel source -----------------------------------------------------------------------
  std::string src = kPrelude;
  auto W = [](int k) { return "W[" + std::to_string(k) + "]"; };
  const int w_v = kWHead, w_n = kWHead + nv, w_h = kWHead + 2 * nv, w_o = kWHead + 2 * nv + nh;
  p.jit_words = w_o + ne;
  // typed views of the W words every kernel starts with
  std::string views = "  const i64 range = (i64)W[0], chunk = (i64)W[1];\n  u64* const trap = (u64*)W[6];\n";
  for (int q = 0; q < nv; ++q) {
    const Ty et = m.vecs[q]->elem;
    const std::string t = et == Ty::Double ? "double" : et == Ty::Bool ? "unsigned char" : "i64";
    views += "  const " + t + "* __restrict__ V" + std::to_string(q) + " = (const " + t + "*)" + W(w_v + q) + ";\n";
    views += "  const i64 N" + std::to_string(q) + " = (i64)" + W(w_n + q) + ";\n";
  }
  for (int h = 0; h < nh; ++h) views += "  const u64 H" + std::to_string(h) + " = " + W(w_h + h) + ";\n";
  for (int q = 0; q < ne; ++q)
    if (p.jit_kind[q] == 1 || p.jit_kind[q] == 2) views += "  void* const O" + std::to_string(q) + " = (void*)" + W(w_o + q) + ";\n";
  views += "  (void)range; (void)chunk; (void)trap;\n";
  const std::string T = std::to_string(kJitThreads);
  const std::string NA = std::to_string(std::max(napp, 1));
  const std::string NR = std::to_string(std::max(nred, 1));

  if (napp) {
    // count pass (append elems' selections per CTA range) and the exclusive scan over CTAs
    src += "extern \"C\" __global__ void __launch_bounds__(" + T + ") dlx_count(const u64* __restrict__ W) {\n" + views;
    src += "  i64* const counts = (i64*)W[3];\n";
    src += "  const i64 lo = (i64)blockIdx.x * chunk, hi = lo + chunk < range ? lo + chunk : range;\n";
    for (int a = 0; a < napp; ++a) src += "  i64 cnt" + std::to_string(a) + " = 0;\n";
    src += "  for (i64 i = lo + threadIdx.x; i < hi; i += " + T + ") {\n    {\n" + count_body + "    }\n    continue;\n  L_trap:;\n  }\n";
    src += "  __shared__ i64 cnt_s[" + NA + "];\n  if (threadIdx.x < " + NA + ") cnt_s[threadIdx.x] = 0;\n  __syncthreads();\n";
    for (int a = 0; a < napp; ++a) {
      const std::string as = std::to_string(a);
      src += "  { i64 v = cnt" + as + "; for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);\n"
             "    if ((threadIdx.x & 31) == 0) atomicAdd((u64*)&cnt_s[" + as + "], (u64)v); }\n";
    }
    src += "  __syncthreads();\n  if (threadIdx.x < " + NA + ") counts[(i64)blockIdx.x * " + NA + " + threadIdx.x] = cnt_s[threadIdx.x];\n}\n";
    src += "extern \"C\" __global__ void dlx_scan(const u64* __restrict__ W, int nblocks) {\n"
           "  const i64* counts = (const i64*)W[3]; i64* offsets = (i64*)W[4]; u64* res = (u64*)W[5];\n"
           "  const int a = threadIdx.x;\n  if (a >= " + NA + ") return;\n  i64 run = 0;\n"
           "  for (int b = 0; b < nblocks; ++b) { offsets[(i64)b * " + NA + " + a] = run; run += counts[(i64)b * " + NA + " + a]; }\n";
    for (int q = 0; q < ne; ++q)
      if (p.jit_kind[q] == 2) src += "  if (a == " + std::to_string(app_of[q]) + ") res[" + std::to_string(q) + "] = (u64)run;\n";
    src += "}\n";
  }

  // main pass
  src += "extern \"C\" __global__ void __launch_bounds__(" + T + ") dlx_main(const u64* __restrict__ W) {\n" + views;
  src += "  u64* const parts = (u64*)W[2];\n  const i64* const offsets = (const i64*)W[4];\n  (void)offsets; (void)parts;\n";
  src += "  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;\n  (void)lane; (void)warp;\n";
  for (int q = 0; q < ne; ++q)
    if (p.jit_kind[q] == 0) {
      // start at the combine's identity (-0.0 + x == x for every x); the zero is folded once
      const std::string id = ety[q] == Ty::Double ? (comb[q] ? "1.0" : "-0.0") : (comb[q] ? "(i64)1" : "(i64)0");
      src += "  " + ctype(ety[q]) + " acc" + std::to_string(red_of[q]) + " = " + id + ";\n";
    }
  for (int q = 0; q < ne; ++q)
    if (p.jit_kind[q] == 2) {
      const std::string a = std::to_string(app_of[q]);
      src += "  i64 run" + a + " = offsets[(i64)blockIdx.x * " + NA + " + " + a + "];\n";
    }
  if (napp) {
    src += "  __shared__ int wsum_s[" + std::to_string(kJitThreads / 32) + "];\n";
    src += "  i64 i0, stop, step;\n  { i0 = (i64)blockIdx.x * chunk; stop = i0 + chunk < range ? i0 + chunk : range; step = " + T + "; }\n";
  } else {
    src += "  const i64 i0 = (i64)blockIdx.x * " + T + ", stop = range, step = (i64)gridDim.x * " + T + ";\n";
  }
  src += "  for (i64 base = i0; base < stop; base += step) {\n    const i64 i = base + threadIdx.x;\n";
  for (int q = 0; q < ne; ++q)
    if (p.jit_kind[q] == 2) {
      const std::string a = std::to_string(app_of[q]);
      src += "    bool tk" + a + " = false; " + (ety[q] == Ty::Bool ? std::string("bool") : ctype(ety[q])) + " av" + a + "{};\n";
    }
  src += "    if (i < stop) {\n      {\n" + main_body + "      }\n      goto L_done;\n    L_trap:;\n";
  for (int q = 0; q < ne; ++q)
    if (p.jit_kind[q] == 2) src += "      tk" + std::to_string(app_of[q]) + " = false;\n";
  src += "    L_done:;\n    }\n";
  for (int q = 0; q < ne; ++q)
    if (p.jit_kind[q] == 2) {   // block-uniform: every thread reaches the ordered compaction
      const std::string a = std::to_string(app_of[q]), qs = std::to_string(q);
      const std::string store = ety[q] == Ty::Bool ? "((unsigned char*)O" + qs + ")[at] = (unsigned char)(av" + a + " ? 1 : 0);"
                                                   : "((" + ctype(ety[q]) + "*)O" + qs + ")[at] = av" + a + ";";
      src += "    { const unsigned bal = __ballot_sync(0xffffffffu, tk" + a + ");\n"
             "      if (lane == 0) wsum_s[warp] = __popc(bal);\n      __syncthreads();\n"
             "      int before = 0, total = 0;\n"
             "      for (int w = 0; w < " + std::to_string(kJitThreads / 32) + "; ++w) { const int c = wsum_s[w]; before += w < warp ? c : 0; total += c; }\n"
             "      if (tk" + a + ") { const i64 at = run" + a + " + before + __popc(bal & ((1u << lane) - 1)); " + store + " }\n"
             "      run" + a + " += total;\n      __syncthreads(); }\n";
    }
  src += "  }\n";
  if (nred) {
    // warp tree, then ascending-warp fold, kFoldChunk reduce elems per shared-memory round
    src += "  __shared__ u64 red_s[" + std::to_string(kJitThreads / 32) + "][" + std::to_string(kFoldChunk) + "];\n";
    for (int c0 = 0; c0 < nred; c0 += kFoldChunk) {
      const int c1 = std::min(nred, c0 + kFoldChunk);
      for (int q = 0; q < ne; ++q) {
        const int r = red_of[q];
        if (r < c0 || r >= c1) continue;
        const std::string rs = std::to_string(r);
        src += "  { " + ctype(ety[q]) + " v = acc" + rs + "; for (int o = 16; o > 0; o >>= 1) v = " +
               (comb[q] ? "cmul" : "cadd") + "(v, shfl(v, o));\n    if (lane == 0) red_s[warp][" + std::to_string(r - c0) + "] = tobits(v); }\n";
      }
      src += "  __syncthreads();\n";
      for (int q = 0; q < ne; ++q) {
        const int r = red_of[q];
        if (r < c0 || r >= c1) continue;
        const std::string rs = std::to_string(r);
        src += "  if (threadIdx.x == " + std::to_string(r - c0) + ") { " + ctype(ety[q]) + " v, u; frombits(red_s[0][" +
               std::to_string(r - c0) + "], v);\n    for (int w = 1; w < " + std::to_string(kJitThreads / 32) +
               "; ++w) { frombits(red_s[w][" + std::to_string(r - c0) + "], u); v = " + (comb[q] ? "cmul" : "cadd") +
               "(v, u); }\n    parts[(i64)blockIdx.x * " + NR + " + " + rs + "] = tobits(v); }\n";
      }
      src += "  __syncthreads();\n";
    }
    // final: the elem's zero, then the CTA partials in ascending order (one thread per reduce)
    src += "}\nextern \"C\" __global__ void dlx_final(const u64* __restrict__ W, int nparts) {\n"
           "  const u64* parts = (const u64*)W[2]; u64* res = (u64*)W[5];\n  const int r = blockIdx.x * blockDim.x + threadIdx.x;\n";
    for (int q = 0; q < ne; ++q) {
      if (p.jit_kind[q] != 0) continue;
      const LElem& le = els[q];
      uint64_t zb = static_cast<uint64_t>(le.e->zero.i);
      if (le.e->zero.k == Atom::Double) std::memcpy(&zb, &le.e->zero.d, 8);
      if (ety[q] == Ty::Double && le.e->zero.k == Atom::Int) {   // an Int literal zero of a Double reduce
        const double zd = static_cast<double>(le.e->zero.i);
        std::memcpy(&zb, &zd, 8);
      }
      const std::string rs = std::to_string(red_of[q]);
      src += "  if (r == " + rs + ") { " + ctype(ety[q]) + " v, u; frombits(" + hex64(zb) + ", v);\n"
             "    for (int b = 0; b < nparts; ++b) { frombits(parts[(i64)b * " + NR + " + " + rs + "], u); v = " +
             (comb[q] ? "cmul" : "cadd") + "(v, u); }\n    res[" + std::to_string(q) + "] = tobits(v); }\n";
    }
  }
  src += "}\n";
  p.jit_src = std::move(src);
  p.jit_names = {"dlx_main"};
  if (nred) p.jit_names.push_back("dlx_final");
  if (napp) {
    p.jit_names.push_back("dlx_count");
    p.jit_names.push_back("dlx_scan");
  }
  if (const char* dir = getenv("DLX_JIT_DUMP")) {   // the generated source, for inspection
    static int seq = 0;
    const std::string path = std::string(dir) + "/multiloop_" + std::to_string(seq++) + ".cu";
    if (FILE* f = fopen(path.c_str(), "w")) {
      fwrite(p.jit_src.data(), 1, p.jit_src.size(), f);
      fclose(f);
    }
  }
  if (g_run->dry) {
    // dry run: the source is generated and compiled (NVRTC needs no device), never loaded
    if (getenv("DLX_PROGRAM_DRYRUN_COMPILE")) jit_check(p.jit_src);
  }
  p.fam = LoopPlan::Compiled;
  p.family = "compiled";
  p.launch = "nvrtc:dlx_main";
  p.nres = ne + 1;
  return true;
}

static int jit_grid(int64_t range) {
  int sms = 148;
  dlx_sm_count(&sms);
  const int64_t need = (range + kJitThreads - 1) / kJitThreads;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, static_cast<int64_t>(sms) * 4)));
}

void Executor::launch_compiled(LoopPlan& p, int64_t n, std::vector<VecP>& V) {
  wait_inputs(V);
  if (!p.jit) p.jit = jit_compile(p.jit_src, p.jit_names);
  const JitModule& mod = *p.jit;
  const int ne = static_cast<int>(p.jit_kind.size());
  const int nv = static_cast<int>(V.size());
  const int nh = static_cast<int>(p.jit_host.size());
  const int grid = jit_grid(n);
  const int na = std::max(p.jit_napp, 1), nr = std::max(p.jit_nred, 1);
  std::vector<VecP> outs(ne);
  for (int q = 0; q < ne; ++q)
    if (p.jit_kind[q] != 0) outs[q] = new_vec(n, p.coll_ty[q], lst_, true);
  // one device block: W words, result record (+ trap word), CTA partials, append counts/offsets
  const size_t wbytes = static_cast<size_t>(p.jit_words) * 8, rbytes = static_cast<size_t>(ne + 1) * 8;
  const size_t pbytes = static_cast<size_t>(grid) * nr * 8, abytes = static_cast<size_t>(grid) * na * 8;
  auto* blk = static_cast<unsigned char*>(dalloc(wbytes + rbytes + pbytes + 2 * abytes));
  uint64_t* dW = reinterpret_cast<uint64_t*>(blk);
  uint64_t* dres = reinterpret_cast<uint64_t*>(blk + wbytes);
  unsigned char* dparts = blk + wbytes + rbytes;
  unsigned char* dcounts = dparts + pbytes;
  unsigned char* doffsets = dcounts + abytes;
  const int64_t chunk = p.jit_napp ? (n + grid - 1) / grid : 0;
  // W and the initial result record (zeros; trap word UINT64_MAX) staged through pinned memory
  auto* hW = res_->pin.get_n<uint64_t>(p.jit_words + ne + 1);
  uint64_t* hres0 = hW + p.jit_words;
  auto u = [](const void* ptr) { return static_cast<uint64_t>(reinterpret_cast<uintptr_t>(ptr)); };
  hW[kWRange] = static_cast<uint64_t>(n);
  hW[kWChunk] = static_cast<uint64_t>(chunk);
  hW[kWParts] = u(dparts);
  hW[kWCounts] = u(dcounts);
  hW[kWOffsets] = u(doffsets);
  hW[kWRes] = u(dres);
  hW[kWTrap] = u(dres + ne);
  for (int q = 0; q < nv; ++q) {
    hW[kWHead + q] = u(V[q]->p);
    hW[kWHead + nv + q] = static_cast<uint64_t>(V[q]->n);
  }
  for (int h = 0; h < nh; ++h) hW[kWHead + 2 * nv + h] = static_cast<uint64_t>(val_bits_of(force(env_[p.jit_host[h]])));
  for (int q = 0; q < ne; ++q) hW[kWHead + 2 * nv + nh + q] = outs[q] ? u(outs[q]->p) : 0;
  for (int q = 0; q < ne; ++q) hres0[q] = 0;
  hres0[ne] = ~0ull;
  ckc(cudaMemcpyAsync(dW, hW, wbytes + rbytes, cudaMemcpyHostToDevice, lst_), "cudaMemcpyAsync");
  const uint64_t* wp = dW;
  void* a1[] = {&wp};
  int nb = grid;
  void* a2[] = {&wp, &nb};
  if (p.jit_napp) {
    ckc(cudaLaunchKernel(reinterpret_cast<const void*>(mod.kernels[p.jit_nred ? 2 : 1]), dim3(grid), dim3(kJitThreads),
                         a1, 0, lst_), "jit dlx_count");
    count_launch();
    ckc(cudaLaunchKernel(reinterpret_cast<const void*>(mod.kernels[p.jit_nred ? 3 : 2]), dim3(1), dim3(32 * ((na + 31) / 32)),
                         a2, 0, lst_), "jit dlx_scan");
    count_launch();
  }
  ckc(cudaLaunchKernel(reinterpret_cast<const void*>(mod.kernels[0]), dim3(grid), dim3(kJitThreads), a1, 0, lst_), "jit dlx_main");
  count_launch();
  if (p.jit_nred) {
    ckc(cudaLaunchKernel(reinterpret_cast<const void*>(mod.kernels[1]), dim3((nr + 255) / 256), dim3(256), a2, 0, lst_),
        "jit dlx_final");
    count_launch();
  }
  uint64_t* res = res_->pin.get_n<uint64_t>(ne + 1);
  ckc(cudaMemcpyAsync(res, dres, rbytes, cudaMemcpyDeviceToHost, lst_), "cudaMemcpyAsync");
  dfree(blk);
  std::vector<int> out_syms;
  for (const LoopPlan::Out& o : p.outs) out_syms.push_back(o.sym);
  const std::vector<LoopPlan::Out> po = p.outs;
  const std::vector<uint8_t> kind = p.jit_kind;
  complete_loop(out_syms, [this, res, po, outs, kind, ne] {
    const uint64_t htrap = res[ne];
    if (htrap != ~0ull) {   // the first trap in index order, as sequential execution meets it
      const std::string at = " at index " + std::to_string(htrap >> 2);
      if ((htrap & 3) == 1) trap("TrapDivByZero: integer division by zero in a multiloop" + at);
      trap("TrapIndexOutOfBounds: element load out of range in a multiloop" + at);
    }
    for (const LoopPlan::Out& o : po) {
      if (o.src == 1) {
        const VecP& v = outs[o.ix];
        if (kind[o.ix] == 2) v->n = static_cast<int64_t>(res[o.ix]);   // the builder's final length
        bind(o.sym, Val{v});
      } else {
        bind(o.sym, lazy_val(Lazy{nullptr, static_cast<int64_t>(res[o.ix]), o.ty, 8, true}));
      }
    }
  });
}

}  // namespace dlx
