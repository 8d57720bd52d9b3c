// stagekit_dlx.cpp — serialiser from the reference IR (stagekit Graph + Schedule) to the
// executor's multiloop descriptor.  See stagekit_dlx.hpp.  Written against the reference's
// public headers only (proj/include/stagekit/*.hpp).
#include "stagekit_dlx.hpp"

#include <cmath>
#include <json.hpp>
#include <set>

#include "stagekit/node.hpp"

namespace stagekit_dlx {

using namespace stagekit;
using json = nlohmann::ordered_json;

namespace {

// Doubles as JSON numbers, except the non-finite ones the reference's constant folding can
// produce (graph.cpp:211-216: 1.0/0.0 -> inf, 0.0/0.0 -> nan), which JSON cannot hold as
// numbers: those go as the strings "inf", "-inf", "nan", "-nan" (sign bit kept).
json double_json(double v) {
  if (std::isfinite(v)) return json(v);
  if (std::isnan(v)) return json(std::signbit(v) ? "-nan" : "nan");
  return json(v > 0 ? "inf" : "-inf");
}

json expr_json(const Expr& e) {
  json j;
  if (e.is_sym()) {
    j["s"] = e.sym;
  } else if (e.lit.is_int()) {
    j["i"] = e.lit.i();
  } else if (e.lit.is_double()) {
    j["d"] = double_json(e.lit.d());
  } else if (e.lit.is_bool()) {
    j["b"] = e.lit.b();
  } else if (e.lit.is_str()) {
    j["str"] = e.lit.s();
  } else {
    j["u"] = 1;
  }
  j["t"] = e.ty.to_string();
  return j;
}

// statements and blocks are keyed by id in std::map-ordered objects: an ordered_json object
// looks keys up linearly, which made serialising an unfused production-shape program (4,161
// root loops) quadratic
using keyed_json = nlohmann::json;

struct Writer {
  const Graph& g;
  const Schedule& s;
  keyed_json stmts = keyed_json::object();
  keyed_json blocks = keyed_json::object();
  std::set<BlockId> seen;

  void block(BlockId b) {
    if (b == kNoBlock || seen.count(b)) return;
    seen.insert(b);
    const BlockData& bd = g.block(b);
    json jb;
    jb["stmts"] = json::array();
    for (int32_t idx : s.block_stmts(b)) {
      jb["stmts"].push_back(g.stmts()[idx].sym);
      stmt(idx);
    }
    jb["result"] = expr_json(bd.result);
    jb["bound"] = bd.bound;
    blocks[std::to_string(b)] = keyed_json::parse(jb.dump());
  }

  void stmt(int32_t idx) {
    const Statement& st = g.stmts()[idx];
    json js;
    js["op"] = op_name(st.def.op);
    js["ty"] = st.ty.to_string();
    js["args"] = json::array();
    for (const Expr& a : st.def.args) js["args"].push_back(expr_json(a));
    if (!st.def.blocks.empty()) js["blocks"] = st.def.blocks;
    if (!st.def.aux_ty.is(Ty::Unit)) js["aux_ty"] = st.def.aux_ty.to_string();
    if (!st.def.str.empty()) js["str"] = st.def.str;
    if (!st.def.lits.empty()) {
      js["lits"] = json::array();
      for (const Lit& l : st.def.lits) {
        json jl;
        if (l.is_int()) jl["i"] = l.i();
        else if (l.is_double()) jl["d"] = double_json(l.d());
        else if (l.is_bool()) jl["b"] = l.b();
        js["lits"].push_back(jl);
      }
    }
    for (BlockId b : st.def.blocks) block(b);
    if (st.def.loop) {
      const LoopPayload& lp = *st.def.loop;
      json jl;
      jl["range"] = expr_json(lp.range);
      jl["index"] = lp.index_var;
      jl["body"] = lp.body_scope;
      block(lp.body_scope);
      jl["elems"] = json::array();
      for (size_t k = 0; k < lp.elems.size(); ++k) {
        const LoopElem& el = lp.elems[k];
        json je;
        je["kind"] = el.kind == LoopElem::K::Collect ? "collect"
                     : el.kind == LoopElem::K::Reduce ? "reduce"
                                                      : "foreach";
        je["live"] = s.elem_live(idx, k);
        je["out"] = el.out;
        je["out_ty"] = el.out_ty.to_string();
        je["elem"] = el.elem;
        je["cond"] = el.cond;
        je["combine"] = el.combine;
        je["append"] = el.append;
        if (el.kind == LoopElem::K::Reduce) {
          je["zero"] = expr_json(el.zero);
          je["rv_left"] = el.rv_left;
          je["rv_right"] = el.rv_right;
        }
        if (s.elem_live(idx, k)) {
          block(el.elem);
          block(el.cond);
          block(el.combine);
        }
        jl["elems"].push_back(std::move(je));
      }
      js["loop"] = std::move(jl);
    }
    stmts[std::to_string(st.sym)] = keyed_json::parse(js.dump());
  }
};

}  // namespace

std::string to_dlx_program(const Graph& g, const Schedule& s, bool with_deg, bool executor_fusion) {
  Writer w{g, s};
  w.block(g.root());
  std::string out = "{\"format\":\"dlx-program/1\",\"root\":" + std::to_string(g.root());
  // an unfused graph: the executor fuses the root loops itself (csrc/fuse.cpp)
  if (executor_fusion) out += ",\"fusion\":\"executor\"";
  out += ",\"stmts\":" + w.stmts.dump() + ",\"blocks\":" + w.blocks.dump();
  // the DEG exactly as the reference builds it (codegen.cpp:497-588); the executor derives its
  // own order and overlap from the statements, so an unfused production-shape program (whose
  // ordered-effect anti-dependence lists grow quadratically) can leave it out
  if (with_deg) out += ",\"deg\":" + json::parse(deg_to_json(build_kernels(g, s))).dump();
  return out + "}";
}

std::string to_dlx_program_unfused(const Graph& g, const Schedule& s) {
  return to_dlx_program(g, s, /*with_deg=*/false, /*executor_fusion=*/true);
}

}  // namespace stagekit_dlx

