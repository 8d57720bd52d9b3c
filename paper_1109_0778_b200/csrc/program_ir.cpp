// program_ir.cpp — parsing of "dlx-program/1" descriptors and the per-program static analyses
// (see program_ir.hpp).  Runs once per program handle; executions reuse the result.
#include "program_ir.hpp"

#include "fuse.hpp"

#include <charconv>
#include <cmath>
#include <json.hpp>
#include <cstring>
#include <limits>
#include <unordered_set>

namespace dlx {

using json = nlohmann::json;

std::string format_double(double x) {   // expr.cpp:11-22: shortest round trip, ".0" if integral
  if (std::isnan(x)) return "nan";
  if (std::isinf(x)) return x > 0 ? "inf" : "-inf";
  char buf[64];
  auto res = std::to_chars(buf, buf + sizeof(buf), x);
  std::string s(buf, res.ptr);
  if (s.find('.') == std::string::npos && s.find('e') == std::string::npos) s += ".0";
  return s;
}

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

Op parse_op(const std::string& s) {
  static const std::unordered_map<std::string, Op> ops = {
      {"Plus", Op::Plus}, {"Minus", Op::Minus}, {"Times", Op::Times}, {"Divide", Op::Divide},
      {"Lt", Op::Lt}, {"Eq", Op::Eq}, {"And", Op::And}, {"Or", Op::Or}, {"Not", Op::Not},
      {"MathAbs", Op::MathAbs}, {"MathSqrt", Op::MathSqrt}, {"MathExp", Op::MathExp},
      {"ToDouble", Op::ToDouble}, {"IfThenElse", Op::IfThenElse}, {"While", Op::While},
      {"VarAlloc", Op::VarAlloc}, {"VarRead", Op::VarRead}, {"VarWrite", Op::VarWrite},
      {"Print", Op::Print}, {"VectorNew", Op::VectorNew}, {"VectorRand", Op::VectorRand},
      {"VectorRandInt", Op::VectorRandInt}, {"VectorLiteral", Op::VectorLiteral},
      {"VectorLength", Op::VectorLength}, {"VectorApply", Op::VectorApply},
      {"VectorUpdate", Op::VectorUpdate}, {"ParallelLoop", Op::ParallelLoop}};
  auto it = ops.find(s);
  return it == ops.end() ? Op::Unknown : it->second;
}

namespace {

// a Double literal: a JSON number, or "inf" / "-inf" / "nan" / "-nan" for the non-finite values
// the reference's constant folding produces (graph.cpp:211-216), which JSON numbers cannot hold
// (integration/stagekit_dlx.cpp writes them so)
double json_double(const json& v) {
  if (!v.is_string()) return v.get<double>();
  const std::string& s = v.get_ref<const std::string&>();
  if (s == "inf") return INFINITY;
  if (s == "-inf") return -INFINITY;
  if (s == "nan") return std::copysign(std::numeric_limits<double>::quiet_NaN(), 1.0);
  if (s == "-nan") return std::copysign(std::numeric_limits<double>::quiet_NaN(), -1.0);
  throw Fail(DLX_ERR_ARG, "malformed Double literal: " + s);
}

Atom parse_atom(const json& j) {
  Atom a;
  if (j.contains("t")) a.ty = parse_type(j["t"].get<std::string>());
  if (j.contains("s")) a.k = Atom::Sym, a.sym = j["s"].get<int>();
  else if (j.contains("i")) a.k = Atom::Int, a.i = j["i"].get<int64_t>();
  else if (j.contains("d")) a.k = Atom::Double, a.d = json_double(j["d"]);
  else if (j.contains("b")) a.k = Atom::Bool, a.b = j["b"].get<bool>();
  else if (j.contains("str")) a.k = Atom::Str, a.s = j["str"].get<std::string>();
  return a;
}

// ---- analyses ---------------------------------------------------------------------------------
struct Analyzer {
  Program& P;
  std::vector<int32_t> print_uses;

  void use(const Atom& a, bool print) {
    if (a.k != Atom::Sym || a.sym < 0 || a.sym > P.max_sym) return;
    ++P.uses[a.sym];
    if (print) ++print_uses[a.sym];
  }

  void count_uses() {
    P.uses.assign(P.max_sym + 1, 0);
    print_uses.assign(P.max_sym + 1, 0);
    for (const Stmt& s : P.stmts) {
      if (s.sym < 0) continue;
      for (const Atom& a : s.args) use(a, s.op == Op::Print);
      if (s.loop) {
        use(s.loop->range, false);
        for (const Elem& e : s.loop->elems)
          if (e.live && e.kind == Elem::Reduce) use(e.zero, false);
      }
    }
    for (size_t b = 0; b < P.blocks.size(); ++b)
      if (P.has_block[b]) use(P.blocks[b].result, false);
    P.print_only.assign(P.max_sym + 1, 0);
    for (int s = 0; s <= P.max_sym; ++s) P.print_only[s] = P.uses[s] > 0 && P.uses[s] == print_uses[s];
  }

  // every symbol a statement reads, including inside its nested blocks (IfThenElse / While
  // bodies, loop blocks)
  void refs_block(int b, std::unordered_set<int>& out, int depth) {
    if (b < 0 || b >= static_cast<int>(P.blocks.size()) || !P.has_block[b] || depth > 64) return;
    const Block& bl = P.blocks[b];
    for (int s : bl.stmts) refs_stmt(P.stmts[s], out, depth + 1);
    if (bl.result.k == Atom::Sym) out.insert(bl.result.sym);
  }
  void refs_stmt(const Stmt& s, std::unordered_set<int>& out, int depth) {
    for (const Atom& a : s.args)
      if (a.k == Atom::Sym) out.insert(a.sym);
    for (int b : s.blocks) refs_block(b, out, depth);
    if (s.loop) {
      if (s.loop->range.k == Atom::Sym) out.insert(s.loop->range.sym);
      refs_block(s.loop->body, out, depth);
      for (const Elem& e : s.loop->elems) {
        if (!e.live) continue;
        refs_block(e.elem, out, depth);
        refs_block(e.cond, out, depth);
        refs_block(e.combine, out, depth);
      }
    }
  }

  void find_copy_runs() {
    for (size_t b = 0; b < P.blocks.size(); ++b) {
      if (!P.has_block[b]) continue;
      const std::vector<int>& ss = P.blocks[b].stmts;
      size_t q = 0;
      while (q + 1 < ss.size()) {
        CopyRun run;
        size_t r = q;
        while (r + 1 < ss.size()) {
          const Stmt& a = P.stmts[ss[r]];
          const Stmt& u = P.stmts[ss[r + 1]];
          const bool pair = a.op == Op::VectorApply && a.args.size() == 2 && a.args[0].k == Atom::Sym &&
                            a.args[1].k == Atom::Int && u.op == Op::VectorUpdate && u.args.size() == 3 &&
                            u.args[0].k == Atom::Sym && u.args[1].k == Atom::Int && u.args[2].k == Atom::Sym &&
                            u.args[2].sym == a.sym && P.uses[a.sym] == 1 && a.args[0].sym != u.args[0].sym;
          if (!pair || (run.x_sym >= 0 && (run.x_sym != a.args[0].sym || run.v_sym != u.args[0].sym))) break;
          run.x_sym = a.args[0].sym;
          run.v_sym = u.args[0].sym;
          run.pairs.emplace_back(a.args[1].i, u.args[1].i);
          run.stmts.push_back(a.sym);
          run.stmts.push_back(u.sym);
          r += 2;
        }
        if (run.pairs.size() >= 2) {
          P.copy_runs[ss[q]] = std::move(run);
          q = r;
        } else {
          ++q;
        }
      }
    }
  }

  // UpdateGroups after each loop L (see program_ir.hpp): per target V, the entries and every
  // statement computing them; a group is kept when its temporaries are read only inside it,
  // no other statement touches V before its last update, and (axpy) one alpha serves all.
  void find_update_groups() {
    for (size_t b = 0; b < P.blocks.size(); ++b) {
      if (!P.has_block[b]) continue;
      const std::vector<int>& ss = P.blocks[b].stmts;
      for (size_t p = 0; p < ss.size(); ++p) {
        const Stmt& L = P.stmts[ss[p]];
        if (L.op != Op::ParallelLoop || !L.loop) continue;
        std::unordered_set<int> outs;
        for (const Elem& e : L.loop->elems)
          if (e.live && e.kind == Elem::Reduce) outs.insert(e.out);
        if (outs.empty()) continue;
        auto is_out = [&](const Atom& a) { return a.k == Atom::Sym && outs.count(a.sym); };
        auto is_alpha = [&](const Atom& a) {   // a literal or a host scalar computed before the loop
          return a.k == Atom::Double || (a.k == Atom::Sym && !outs.count(a.sym));
        };
        // candidate temporaries: sym -> defining statement's position
        std::unordered_map<int, int> cd_of;                    // ToDouble(count) -> count
        std::unordered_map<int, std::pair<int, int>> q_of;     // Divide(sum, cd) -> (sum, cd)
        std::unordered_map<int, std::pair<int, Atom>> t_of;    // Times(alpha, g) -> (g, alpha)
        std::unordered_map<int, std::pair<int, int64_t>> a_of; // VectorApply(V, j) -> (V, j)
        std::unordered_map<int, std::pair<int, int>> m_of;     // Minus(a, t) -> (a, t)
        struct Cand {
          UpdateGroup g;
          size_t last = 0;
          bool mixed_alpha = false;
          bool has_alpha = false;
          Atom alpha;
        };
        std::unordered_map<int, Cand> cands[2];   // [Div, Axpy] by V
        std::vector<int> pos_of_sym;               // position of each candidate statement
        std::unordered_map<int, size_t> pos;
        for (size_t q = p + 1; q < ss.size(); ++q) {
          const Stmt& s = P.stmts[ss[q]];
          pos[s.sym] = q;
          const auto& A = s.args;
          if (s.op == Op::ToDouble && A.size() == 1 && is_out(A[0])) cd_of[s.sym] = A[0].sym;
          else if (s.op == Op::Divide && A.size() == 2 && is_out(A[0]) && A[1].k == Atom::Sym && cd_of.count(A[1].sym))
            q_of[s.sym] = {A[0].sym, A[1].sym};
          else if (s.op == Op::Times && A.size() == 2 && is_out(A[1]) && is_alpha(A[0])) t_of[s.sym] = {A[1].sym, A[0]};
          else if (s.op == Op::Times && A.size() == 2 && is_out(A[0]) && is_alpha(A[1])) t_of[s.sym] = {A[0].sym, A[1]};
          else if (s.op == Op::VectorApply && A.size() == 2 && A[0].k == Atom::Sym && A[1].k == Atom::Int)
            a_of[s.sym] = {A[0].sym, A[1].i};
          else if (s.op == Op::Minus && A.size() == 2 && A[0].k == Atom::Sym && A[1].k == Atom::Sym && a_of.count(A[0].sym) &&
                   t_of.count(A[1].sym))
            m_of[s.sym] = {A[0].sym, A[1].sym};
          else if (s.op == Op::VectorUpdate && A.size() == 3 && A[0].k == Atom::Sym && A[1].k == Atom::Int && A[2].k == Atom::Sym) {
            const int V = A[0].sym;
            const int64_t e = A[1].i;
            if (q_of.count(A[2].sym)) {   // V(e) = sum / toDouble(count)
              const auto [sum, cd] = q_of[A[2].sym];
              Cand& c = cands[UpdateGroup::Div][V];
              c.g.kind = UpdateGroup::Div;
              c.g.vec_sym = V;
              c.g.entries.push_back({e, sum, cd_of[cd]});
              c.g.stmts.insert(c.g.stmts.end(), {s.sym, A[2].sym});
              c.last = q;
            } else if (m_of.count(A[2].sym)) {   // V(e) = V(e) - alpha * g
              const auto [a, t] = m_of[A[2].sym];
              if (a_of[a].first != V || a_of[a].second != e) continue;
              Cand& c = cands[UpdateGroup::Axpy][V];
              c.g.kind = UpdateGroup::Axpy;
              c.g.vec_sym = V;
              c.g.entries.push_back({e, t_of[t].first, -1});
              c.g.stmts.insert(c.g.stmts.end(), {s.sym, A[2].sym, a, t});
              const Atom& al = t_of[t].second;
              if (!c.has_alpha) {
                c.alpha = al;
                c.has_alpha = true;
              } else if (al.k != c.alpha.k || (al.k == Atom::Sym ? al.sym != c.alpha.sym : std::memcmp(&al.d, &c.alpha.d, 8) != 0)) {
                c.mixed_alpha = true;
              }
              c.last = q;
            }
          }
        }
        UpdateGroup best;
        for (int kind = 0; kind < 2; ++kind)
          for (auto& [V, c] : cands[kind]) {
            if (c.mixed_alpha || c.g.entries.size() <= best.entries.size()) continue;
            UpdateGroup g = c.g;
            if (kind == UpdateGroup::Div) {   // the ToDouble temporaries join the group
              std::unordered_set<int> cds;
              for (int st : c.g.stmts)
                if (q_of.count(st)) cds.insert(q_of[st].second);
              g.stmts.insert(g.stmts.end(), cds.begin(), cds.end());
            }
            std::unordered_set<int> in(g.stmts.begin(), g.stmts.end());
            // every temporary is read only by statements of the group
            bool ok = true;
            for (int st : g.stmts) {
              const Stmt& S = P.stmts[st];
              if (S.op == Op::VectorUpdate) continue;
              int inside = 0;
              for (int u : g.stmts)
                for (const Atom& a : P.stmts[u].args)
                  if (a.k == Atom::Sym && a.sym == st) ++inside;
              if (P.uses[st] != inside) ok = false;
            }
            // nothing outside the group touches V before its last update
            for (size_t q = p + 1; q <= c.last && ok; ++q) {
              if (in.count(ss[q])) continue;
              std::unordered_set<int> r;
              refs_stmt(P.stmts[ss[q]], r, 0);
              if (r.count(V)) ok = false;
            }
            if (!ok) continue;
            if (kind == UpdateGroup::Axpy) g.alpha = c.alpha;
            best = std::move(g);
          }
        if (!best.entries.empty()) P.update_after[L.sym] = std::move(best);
      }
    }
  }
};

}  // namespace

std::shared_ptr<Program> parse_program(const char* text, size_t len) {
  json j = json::parse(text, text + len);
  if (j.value("format", "") != "dlx-program/1") throw Fail(DLX_ERR_ARG, "not a dlx-program/1 descriptor");
  auto pp = std::make_shared<Program>();
  Program& p = *pp;
  p.root = j["root"].get<int>();
  int max_sym = -1, max_block = p.root;
  auto see = [&](int s) { max_sym = std::max(max_sym, s); };
  for (auto& [k, v] : j["blocks"].items()) {
    max_block = std::max(max_block, std::stoi(k));
    if (v.contains("bound"))
      for (auto& b : v["bound"]) see(b.get<int>());
  }
  for (auto& [k, v] : j["stmts"].items()) {
    see(std::stoi(k));
    if (v.contains("loop")) {
      const json& jl = v["loop"];
      see(jl["index"].get<int>());
      for (auto& je : jl["elems"]) {
        see(je["out"].get<int>());
        see(je.value("rv_left", -1));
        see(je.value("rv_right", -1));
      }
    }
  }
  if (max_sym > (1 << 28) || max_block > (1 << 28)) throw Fail(DLX_ERR_ARG, "descriptor symbols out of range");
  p.max_sym = max_sym;
  p.stmts.resize(max_sym + 1);
  p.blocks.resize(max_block + 1);
  p.has_block.assign(max_block + 1, 0);
  for (auto& [k, v] : j["blocks"].items()) {
    const int id = std::stoi(k);
    Block& b = p.blocks[id];
    for (auto& s : v["stmts"]) b.stmts.push_back(s.get<int>());
    b.result = parse_atom(v["result"]);
    p.has_block[id] = 1;
  }
  for (auto& [k, v] : j["stmts"].items()) {
    Stmt& s = p.stmts[std::stoi(k)];
    s.sym = std::stoi(k);
    s.opname = v["op"].get<std::string>();
    s.op = parse_op(s.opname);
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
        const std::string kind = je["kind"].get<std::string>();
        e.kind = kind == "collect" ? Elem::Collect : kind == "reduce" ? Elem::Reduce : Elem::Foreach;
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
  }
  // every statement a block lists must exist
  for (size_t b = 0; b < p.blocks.size(); ++b)
    if (p.has_block[b])
      for (int s : p.blocks[b].stmts) p.stmt(s);
  p.block(p.root);
  // an unfused graph (the adapter skipped the reference's fuse_loops): fuse here, before the
  // analyses, so update groups and copy runs see the fused loops
  if (j.value("fusion", "") == "executor") p.fused_pairs = fuse_loops_linear(p);
  Analyzer an{p, {}};
  an.count_uses();
  an.find_update_groups();
  an.find_copy_runs();
  return pp;
}

}  // namespace dlx
