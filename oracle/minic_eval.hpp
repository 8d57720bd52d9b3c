// minic_eval.hpp — CPU ORACLE (test infrastructure only): a sequential evaluator for the
// reference's emitted MiniC programs (stagekit::minic::Program, proj/include/stagekit/
// minic.hpp:12-96).  It restates the interpreter the reference declares but does not ship,
//     RunResult interpret(const minic::Program&, uint64_t seed)      (interp.hpp:10)
// with the semantics of SPEC.md:635-643 and the builtins of default_emitters
// (proj/src/codegen.cpp:437-481):
//   randVector(n)        n next_unit() draws of one shared Rng(seed), in execution order
//   randIntVector(n, b)  n next_int(b) draws of the same Rng                (runtime.hpp:86-96)
//   length / new_array#T(n) (zero-filled) / new_builder#T() / array#T(...) / toDouble / abs / sqrt
// Int arithmetic wraps (graph.cpp:10-21), Int division by zero traps, Double is IEEE,
// array reads and writes are bounds-checked (TrapIndexOutOfBounds), println uses
// format_double for doubles (expr.cpp:11-22).  Names are resolved to slots once, so evaluating
// the C1 k-means program (10 unrolled-equivalent iterations) takes seconds, not minutes.
#pragma once

#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <variant>
#include <vector>

#include "stagekit/errors.hpp"
#include "stagekit/expr.hpp"
#include "stagekit/minic.hpp"
#include "stagekit/runtime.hpp"

namespace oracle_minic {

namespace mc = stagekit::minic;

struct Arr;
using ArrPtr = std::shared_ptr<Arr>;
struct V {
  std::variant<std::monostate, int64_t, double, bool, std::string, ArrPtr> v;
  int64_t i() const { return std::get<int64_t>(v); }
  double d() const { return std::get<double>(v); }
  bool b() const { return std::get<bool>(v); }
};
struct Arr {
  std::vector<V> xs;
};

struct EvalResult {
  std::string output;
  V result;
};

class Evaluator {
 public:
  explicit Evaluator(uint64_t seed) : rng_(seed) {}

  EvalResult run(const mc::Program& p) {
    for (const auto& s : p.stmts) {
      if (exec(*s)) break;
    }
    return {out_, ret_};
  }

  static std::string format(const V& x) {
    if (auto p = std::get_if<int64_t>(&x.v)) return std::to_string(*p);
    if (auto p = std::get_if<double>(&x.v)) return stagekit::format_double(*p);
    if (auto p = std::get_if<bool>(&x.v)) return *p ? "true" : "false";
    if (auto p = std::get_if<std::string>(&x.v)) return *p;
    if (auto p = std::get_if<ArrPtr>(&x.v)) {
      std::string s = "[";
      for (size_t k = 0; k < (*p)->xs.size(); ++k) s += (k ? ", " : "") + format((*p)->xs[k]);
      return s + "]";
    }
    return "()";
  }

 private:
  stagekit::Rng rng_;
  std::unordered_map<std::string, size_t> slot_of_;
  std::vector<V> slots_;
  std::string out_;
  V ret_;

  V& slot(const std::string& n) {
    auto it = slot_of_.find(n);
    if (it == slot_of_.end()) {
      it = slot_of_.emplace(n, slots_.size()).first;
      slots_.emplace_back();
    }
    return slots_[it->second];
  }

  [[noreturn]] static void trap(stagekit::TrapError::Kind k, const std::string& m) {
    throw stagekit::TrapError(k, m);
  }

  static ArrPtr arr(const V& a) { return std::get<ArrPtr>(a.v); }
  static int64_t wrap(uint64_t x) { return static_cast<int64_t>(x); }

  V binary(const std::string& op, const V& a, const V& b) {
    if (op == "&&") return {a.b() && b.b()};
    if (op == "||") return {a.b() || b.b()};
    if (std::holds_alternative<int64_t>(a.v) && std::holds_alternative<int64_t>(b.v)) {
      const int64_t x = a.i(), y = b.i();
      if (op == "+") return {wrap(static_cast<uint64_t>(x) + static_cast<uint64_t>(y))};
      if (op == "-") return {wrap(static_cast<uint64_t>(x) - static_cast<uint64_t>(y))};
      if (op == "*") return {wrap(static_cast<uint64_t>(x) * static_cast<uint64_t>(y))};
      if (op == "/") {
        if (y == 0) trap(stagekit::TrapError::Kind::DivByZero, "integer division by zero");
        if (x == INT64_MIN && y == -1) return {x};
        return {x / y};
      }
      if (op == "<") return {x < y};
      if (op == "==") return {x == y};
    }
    if (std::holds_alternative<double>(a.v)) {
      const double x = a.d(), y = b.d();
      if (op == "+") return {x + y};
      if (op == "-") return {x - y};
      if (op == "*") return {x * y};
      if (op == "/") return {x / y};
      if (op == "<") return {x < y};
      if (op == "==") return {x == y};
    }
    if (op == "==") return {a.v == b.v};
    throw std::runtime_error("minic eval: bad binary " + op);
  }

  V call(const mc::Expr& e) {
    const std::string& fn = e.fn;
    std::vector<V> a;
    a.reserve(e.args.size());
    for (const auto& x : e.args) a.push_back(eval(*x));
    if (fn == "randVector") {
      auto r = std::make_shared<Arr>();
      r->xs.resize(static_cast<size_t>(a[0].i()));
      for (auto& x : r->xs) x = V{rng_.next_unit()};
      return {r};
    }
    if (fn == "randIntVector") {
      auto r = std::make_shared<Arr>();
      r->xs.resize(static_cast<size_t>(a[0].i()));
      for (auto& x : r->xs) x = V{rng_.next_int(a[1].i())};
      return {r};
    }
    if (fn == "length") return {static_cast<int64_t>(arr(a[0])->xs.size())};
    if (fn == "toDouble") return {static_cast<double>(a[0].i())};
    if (fn == "sqrt") return {std::sqrt(a[0].d())};
    if (fn == "abs") {
      if (std::holds_alternative<int64_t>(a[0].v)) {
        const int64_t x = a[0].i();
        return {x < 0 ? wrap(0ull - static_cast<uint64_t>(x)) : x};
      }
      return {std::fabs(a[0].d())};
    }
    if (fn.rfind("new_array#", 0) == 0) {
      auto r = std::make_shared<Arr>();
      const std::string t = fn.substr(10);
      V z = t == "Double" ? V{0.0} : t == "Boolean" ? V{false} : V{int64_t{0}};
      r->xs.assign(static_cast<size_t>(a[0].i()), z);
      return {r};
    }
    if (fn.rfind("new_builder#", 0) == 0) return {std::make_shared<Arr>()};
    if (fn.rfind("array#", 0) == 0) {
      auto r = std::make_shared<Arr>();
      r->xs = a;
      return {r};
    }
    throw stagekit::StagingError(stagekit::StagingError::Kind::GenerationFailed,
                                 "minic eval: unknown builtin " + fn);
  }

  V eval(const mc::Expr& e) {
    using K = mc::Expr::K;
    switch (e.k) {
      case K::IntLit: return {e.i};
      case K::DoubleLit: return {e.d};
      case K::BoolLit: return {e.b};
      case K::StrLit: return {e.s};
      case K::UnitLit: return {};
      case K::Ref: return slot(e.s);
      case K::Unary: {
        V a = eval(*e.args[0]);
        if (e.fn == "!") return {!a.b()};
        if (std::holds_alternative<int64_t>(a.v)) return {wrap(0ull - static_cast<uint64_t>(a.i()))};
        return {-a.d()};
      }
      case K::Binary: return binary(e.fn, eval(*e.args[0]), eval(*e.args[1]));
      case K::Call: return call(e);
      case K::Index: {
        V a = eval(*e.args[0]);
        const int64_t i = eval(*e.args[1]).i();
        auto p = arr(a);
        if (i < 0 || i >= static_cast<int64_t>(p->xs.size()))
          trap(stagekit::TrapError::Kind::IndexOutOfBounds, "index " + std::to_string(i));
        return p->xs[static_cast<size_t>(i)];
      }
      case K::Cond: return eval(*e.args[0]).b() ? eval(*e.args[1]) : eval(*e.args[2]);
      default: throw std::runtime_error("minic eval: records are out of scope");
    }
  }

  // returns true on Return
  bool exec(const mc::Stmt& s) {
    using K = mc::Stmt::K;
    switch (s.k) {
      case K::Val:
      case K::Var:
      case K::Assign: slot(s.name) = eval(*s.a); return false;
      case K::Store: {
        auto p = arr(slot(s.name));
        const int64_t i = eval(*s.a).i();
        if (i < 0 || i >= static_cast<int64_t>(p->xs.size()))
          trap(stagekit::TrapError::Kind::IndexOutOfBounds, "store index " + std::to_string(i));
        p->xs[static_cast<size_t>(i)] = eval(*s.b);
        return false;
      }
      case K::Append: arr(slot(s.name))->xs.push_back(eval(*s.a)); return false;
      case K::If: {
        const auto& body = eval(*s.a).b() ? s.body : s.els;
        for (const auto& t : body)
          if (exec(*t)) return true;
        return false;
      }
      case K::While:
        while (eval(*s.a).b())
          for (const auto& t : s.body)
            if (exec(*t)) return true;
        return false;
      case K::Print: out_ += format(eval(*s.a)) + "\n"; return false;
      case K::Return: ret_ = eval(*s.a); return true;
    }
    return false;
  }
};

}  // namespace oracle_minic
