// fuse.cpp — the executor's own multiloop fusion pass for descriptors marked
// "fusion": "executor" (an unfused stagekit graph: the adapter skipped the reference's
// fuse_loops).  See fuse.hpp.
//
// What it does is what the reference's fuse_loops does (proj/src/fusion.cpp:170-288): in every
// block, a later ParallelLoop L joins an earlier one A of the same range (horizontal), or of
// range VectorLength(c) for a dense collect output c of A (vertical, fusion.cpp:204-210); L's
// reads of A's collect outputs at L's own index become the producing elem's value
// (contraction), L's index becomes A's, L's body-scope statements join A's and L's elems are
// appended to A's, in order.  One deliberate difference: a vertical pair A -> VectorLength(c) ->
// L fuses here, while the reference's cycle check rejects it — the VectorLength statement is
// an intermediate on a path from A to L (fusion.cpp:229, PairScan::path_avoiding_direct), so its
// vertical rule (fusion.cpp:204-210) can never fire; here the length of a dense collect of A
// is A's range and L's range is re-pointed at it.  How it does it is different: the reference
// clones the whole graph and rebuilds the whole schedule for every fused pair and restarts its
// scan (quadratic: one
// k-means iteration at k = d = 64, 4,160 reduces, did not finish in 25 min), while this pass
// walks each statement list once, keeping per earlier loop the symbols defined and the vectors
// written since it (linear in the program, up to the number of open candidates).
//
// Legality (checked per pair, conservatively):
//   * neither loop has a Foreach elem (effectful disjoint writes) and L's blocks hold no ordered
//     effect (Print, VectorUpdate, VarWrite), no allocation of mutable storage and no random
//     source (the draw order is program order);
//   * L reads no symbol defined by a statement between A and L (L moves up to A) and no vector
//     or variable written between them;
//   * L reads A's outputs only as VectorApply(c, i_L) for a dense (non-append) collect output c
//     of A — the contraction — never A's reduce results (final only after the loop) and never a
//     collect output at another index.
#include "fuse.hpp"

#include <unordered_map>
#include <unordered_set>

namespace dlx {

namespace {

struct Fuser {
  Program& P;
  int pairs = 0;

  bool valid_block(int b) const { return b >= 0 && b < static_cast<int>(P.blocks.size()) && P.has_block[b]; }

  // every block owned by a statement (IfThenElse / While blocks, loop body and elem blocks)
  void stmt_blocks(const Stmt& s, std::vector<int>& out) const {
    for (int b : s.blocks) out.push_back(b);
    if (s.loop) {
      out.push_back(s.loop->body);
      for (const Elem& e : s.loop->elems) {
        out.push_back(e.elem);
        out.push_back(e.cond);
        out.push_back(e.combine);
      }
    }
  }

  // walk every statement nested in block b (depth-first, program order)
  template <class F>
  void walk_block(int b, F&& f, int depth = 0) const {
    if (!valid_block(b) || depth > 256) return;
    for (int s : P.blocks[b].stmts) {
      const Stmt& st = P.stmts[s];
      f(st);
      std::vector<int> bs;
      stmt_blocks(st, bs);
      for (int c : bs) walk_block(c, f, depth + 1);
    }
  }
  template <class F>
  void walk_stmt(const Stmt& st, F&& f) const {
    f(st);
    std::vector<int> bs;
    stmt_blocks(st, bs);
    for (int c : bs) walk_block(c, f, 1);
  }

  // symbols read by a statement (with everything nested in it), symbols it defines (itself,
  // nested statements, loop indices, elem outputs, reduce operands), vectors / vars it writes
  struct Summary {
    std::unordered_set<int> reads, defs, writes;
    bool effects = false, random = false, foreach = false;
  };
  Summary summarize(const Stmt& top) const {
    Summary S;
    auto atom = [&](const Atom& a) {
      if (a.k == Atom::Sym) S.reads.insert(a.sym);
    };
    walk_stmt(top, [&](const Stmt& st) {
      S.defs.insert(st.sym);
      for (const Atom& a : st.args) atom(a);
      if (st.op == Op::VectorUpdate || st.op == Op::VarWrite) {
        S.effects = true;
        if (!st.args.empty() && st.args[0].k == Atom::Sym) S.writes.insert(st.args[0].sym);
      }
      if (st.op == Op::Print) S.effects = true;
      if (st.op == Op::VectorRand || st.op == Op::VectorRandInt) S.random = true;
      // a loop allocating mutable storage is not fusable (fusion.cpp: fusable_loop)
      if (st.op == Op::VectorNew || st.op == Op::VarAlloc) S.effects = true;
      for (int b : st.blocks)
        if (valid_block(b)) atom(P.blocks[b].result);
      if (st.loop) {
        atom(st.loop->range);
        S.defs.insert(st.loop->index);
        if (valid_block(st.loop->body)) atom(P.blocks[st.loop->body].result);
        for (const Elem& e : st.loop->elems) {
          if (e.kind == Elem::Foreach) S.foreach = true;
          S.defs.insert(e.out);
          if (e.rv_left >= 0) S.defs.insert(e.rv_left);
          if (e.rv_right >= 0) S.defs.insert(e.rv_right);
          if (e.kind == Elem::Reduce) atom(e.zero);
          for (int b : {e.elem, e.cond, e.combine})
            if (valid_block(b)) atom(P.blocks[b].result);
        }
      }
    });
    for (int d : S.defs) S.reads.erase(d);   // block-local definitions are not inputs
    return S;
  }

  static bool same_atom(const Atom& a, const Atom& b) {
    if (a.k != b.k) return false;
    switch (a.k) {
      case Atom::Sym: return a.sym == b.sym;
      case Atom::Int: return a.i == b.i;
      case Atom::Bool: return a.b == b.b;
      case Atom::Double: return a.d == b.d;
      default: return false;
    }
  }

  // --- substitution of symbols by atoms inside L ----------------------------------------------
  void subst_atom(Atom& a, const std::unordered_map<int, Atom>& m) const {
    if (a.k != Atom::Sym) return;
    auto it = m.find(a.sym);
    if (it != m.end()) a = it->second;
  }
  void subst_block(int b, const std::unordered_map<int, Atom>& m, const std::unordered_set<int>& drop, int depth = 0) {
    if (!valid_block(b) || depth > 256) return;
    Block& bl = P.blocks[b];
    std::vector<int> keep;
    keep.reserve(bl.stmts.size());
    for (int s : bl.stmts) {
      if (drop.count(s)) continue;
      keep.push_back(s);
      subst_stmt(P.stmts[s], m, drop, depth + 1);
    }
    bl.stmts.swap(keep);
    subst_atom(bl.result, m);
  }
  void subst_stmt(Stmt& st, const std::unordered_map<int, Atom>& m, const std::unordered_set<int>& drop, int depth) {
    for (Atom& a : st.args) subst_atom(a, m);
    for (int b : st.blocks) subst_block(b, m, drop, depth);
    if (st.loop) {
      subst_atom(st.loop->range, m);
      subst_block(st.loop->body, m, drop, depth);
      for (Elem& e : st.loop->elems) {
        if (e.kind == Elem::Reduce) subst_atom(e.zero, m);
        subst_block(e.elem, m, drop, depth);
        subst_block(e.cond, m, drop, depth);
        subst_block(e.combine, m, drop, depth);
      }
    }
  }

  struct Cand {
    int sym;                              // the loop statement A (in this list)
    std::unordered_set<int> defined_after, written_after;
    bool closed = false;                  // a barrier (an unknown effect) since A
  };

  // Try to fuse L into A; on success L's elems and body statements are A's.
  bool try_fuse(Cand& A, Stmt& L, const Summary& SL, const std::unordered_map<int, int>& len_of) {
    Stmt& AS = P.stmts[A.sym];
    Loop& la = *AS.loop;
    Loop& ll = *L.loop;
    // ranges: equal, or L over VectorLength(c) of a dense collect c of A
    bool vertical = false;
    if (!same_atom(la.range, ll.range)) {
      if (ll.range.k != Atom::Sym) return false;
      auto it = len_of.find(ll.range.sym);
      if (it == len_of.end()) return false;
      bool ok = false;
      for (const Elem& e : la.elems)
        if (e.kind == Elem::Collect && !e.append && e.cond < 0 && e.out == it->second) ok = true;
      if (!ok) return false;
      vertical = true;
    }
    // A's outputs: dense collects (contractable), everything else (reduce results, appends)
    std::unordered_map<int, Atom> collect_val;   // collect out -> the elem's value
    std::unordered_set<int> a_outs;
    for (const Elem& e : la.elems) {
      a_outs.insert(e.out);
      // dense unconditional collects only (fusion.cpp: dense_collect_outs)
      if (e.kind == Elem::Collect && !e.append && e.cond < 0 && valid_block(e.elem))
        collect_val[e.out] = P.blocks[e.elem].result;
    }
    // L's reads: nothing defined or written since A (except a vertical range's length symbol)
    for (int r : SL.reads) {
      if (vertical && r == ll.range.sym) continue;
      if (A.defined_after.count(r) || A.written_after.count(r)) return false;
    }
    // every read of an output of A is a contraction VectorApply(c, i_L)
    std::unordered_set<int> drop;
    std::unordered_map<int, Atom> sub;
    bool bad = false;
    std::vector<int> lbs;
    stmt_blocks(L, lbs);
    for (int b : lbs)
      walk_block(b, [&](const Stmt& st) {
        for (size_t q = 0; q < st.args.size(); ++q) {
          const Atom& a = st.args[q];
          if (a.k != Atom::Sym || !a_outs.count(a.sym)) continue;
          const bool contraction = st.op == Op::VectorApply && q == 0 && st.args.size() == 2 &&
                                   st.args[1].k == Atom::Sym && st.args[1].sym == ll.index &&
                                   collect_val.count(a.sym);
          if (!contraction) {
            bad = true;
            continue;
          }
          drop.insert(st.sym);
          sub[st.sym] = collect_val[a.sym];
        }
      });
    if (bad) return false;
    // a contracted value must not be a block result or range of L (it is, after substitution,
    // an ordinary reference to the producing elem's value, so that is fine); A's outputs must
    // not appear as plain atoms in L's block results / zeros
    for (const Elem& e : ll.elems) {
      if (e.kind == Elem::Reduce && e.zero.k == Atom::Sym && a_outs.count(e.zero.sym)) return false;
      for (int b : {e.elem, e.cond, e.combine})
        if (valid_block(b) && P.blocks[b].result.k == Atom::Sym && a_outs.count(P.blocks[b].result.sym) &&
            !sub.count(P.blocks[b].result.sym))
          return false;
    }
    // ---- merge ----
    Atom ia;
    ia.k = Atom::Sym;
    ia.sym = la.index;
    ia.ty.t = Ty::Int;
    sub[ll.index] = ia;
    subst_block(ll.body, sub, drop);
    for (Elem& e : ll.elems) {
      if (e.kind == Elem::Reduce) subst_atom(e.zero, sub);
      subst_block(e.elem, sub, drop);
      subst_block(e.cond, sub, drop);
      subst_block(e.combine, sub, drop);
    }
    if (valid_block(ll.body) && valid_block(la.body)) {
      std::vector<int>& dst = P.blocks[la.body].stmts;
      const std::vector<int>& src = P.blocks[ll.body].stmts;
      dst.insert(dst.end(), src.begin(), src.end());
      P.blocks[ll.body].stmts.clear();
    }
    for (Elem& e : ll.elems) la.elems.push_back(e);
    ll.elems.clear();
    ++pairs;
    return true;
  }

  void fuse_list(int b) {
    std::vector<int> out;
    std::vector<Cand> cands;
    std::unordered_map<int, int> len_of;   // VectorLength statement -> its vector
    const std::vector<int> in = P.blocks[b].stmts;
    for (int s : in) {
      Stmt& st = P.stmts[s];
      if (st.op == Op::VectorLength && st.args.size() == 1 && st.args[0].k == Atom::Sym) len_of[s] = st.args[0].sym;
      const bool loop = st.op == Op::ParallelLoop && st.loop;
      Summary S = summarize(st);
      if (loop && !S.foreach && !S.effects && !S.random) {
        bool fused = false;
        for (Cand& A : cands) {
          if (A.closed) continue;
          if (try_fuse(A, st, S, len_of)) {
            fused = true;
            // L's outputs are now A's: defined at A, not after it (for later candidates they
            // are defined after those, which is where A sits relative to them: after)
            break;
          }
        }
        if (fused) {
          // the statement leaves the list; its outputs are defined at its fusion target, which
          // for every later candidate is "before" (candidates after the target see them as
          // defined after themselves only if the target follows them — it does not: the
          // target precedes every candidate opened after it)
          st.op = Op::Unknown;
          st.opname = "ParallelLoop (fused)";
          st.loop.reset();
          st.args.clear();
          continue;
        }
      }
      // this statement stays: every open candidate sees its definitions and writes
      for (Cand& A : cands) {
        A.defined_after.insert(S.defs.begin(), S.defs.end());
        A.written_after.insert(S.writes.begin(), S.writes.end());
        if (S.foreach) A.closed = true;
      }
      out.push_back(s);
      if (loop && !S.foreach) {
        Cand c;
        c.sym = s;
        cands.push_back(std::move(c));
      }
    }
    P.blocks[b].stmts.swap(out);
  }

  void run() {
    // blocks in id order (the reference's deterministic block order, fusion.cpp:178-183); a
    // block merged into a target earlier in the walk is still visited under its own id
    for (size_t b = 0; b < P.blocks.size(); ++b)
      if (P.has_block[b] && P.blocks[b].stmts.size() >= 2) fuse_list(static_cast<int>(b));
  }
};

}  // namespace

int fuse_loops_linear(Program& p) {
  Fuser f{p};
  f.run();
  return f.pairs;
}

}  // namespace dlx
