// program_ir.hpp — the executor's in-memory form of a "dlx-program/1" descriptor (the scheduled,
// fused stagekit graph serialised by integration/stagekit_dlx.cpp) and the static analyses run
// once per program handle (dlx_program_create): operator codes, symbol use counts, and the
// centroid-update groups that the k-means lowering executes on the device.
//
// Reference types mirrored here: Op (node.hpp:14-48), Expr atoms (expr.hpp), LoopElem /
// LoopPayload (node.hpp:60-81), BlockData (graph.hpp:18-26), Schedule::block_stmts
// (schedule.hpp:14-36: the descriptor lists every scheduled block's statements in order).
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/dlx.h"

namespace dlx {

// ---- errors (mapped to StagingError::GenerationFailed / TrapError at the API) ----------------
struct Fail : std::runtime_error {
  int code;
  Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void gen_fail(const std::string& m) { throw Fail(DLX_ERR_GENERATION, "GenerationFailed: " + m); }
[[noreturn]] inline void trap(const std::string& m) { throw Fail(DLX_ERR_TRAP, m); }

// ---- IR -------------------------------------------------------------------------------------
enum class Ty : uint8_t { Int, Double, Bool, Str, Unit, Vector, Var, Other };
struct Type {
  Ty t = Ty::Unit;
  Ty elem = Ty::Unit;  // Vector / Var payload
};
Type parse_type(const std::string& s);

// the reference Op set (node.hpp:14-48) plus the MathExp extension (logistic regression)
enum class Op : uint8_t {
  Plus, Minus, Times, Divide, Lt, Eq, And, Or, Not, MathAbs, MathSqrt, MathExp, ToDouble,
  IfThenElse, While, VarAlloc, VarRead, VarWrite, Print,
  VectorNew, VectorRand, VectorRandInt, VectorLiteral, VectorLength, VectorApply, VectorUpdate,
  ParallelLoop, Unknown
};
Op parse_op(const std::string& s);

struct Atom {  // stagekit::Expr: a literal or a symbol
  enum K : uint8_t { Sym, Int, Double, Bool, Str, Unit } k = Unit;
  int sym = -1;
  int64_t i = 0;
  double d = 0;
  bool b = false;
  std::string s;
  Type ty;
};

struct Elem {
  enum Kind : uint8_t { Collect, Reduce, Foreach } kind = Reduce;
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
  Op op = Op::Unknown;
  std::string opname;   // for diagnostics (GenerationFailed messages name the reference op)
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

// A run of host statements after a fused k-means loop that update a centroid vector from the
// loop's reduce results:  cd_c = ToDouble(count_c);  q = Divide(sum_cj, cd_c);
// VectorUpdate(V, e, q)  (vectordsl.cpp:90-103: `mu.update(c*d+j, sum/toDouble(count))`).
// Found statically; the lowering checks at match time that (e, sum, count) cover
// e = c*d + j exactly, and then the statements run as one device update fused into the loop's
// combine launch instead of k*d host statements.
//
// Second kind (logistic-regression BGD, the staged `theta.update(j, theta(j) - alpha * g_j)`):
// t = Times(alpha, g);  a = VectorApply(V, e);  m = Minus(a, t);  VectorUpdate(V, e, m), one alpha
// (a literal or a host scalar) for every entry — run as one axpy after the loop's combine.
struct UpdateGroup {
  enum Kind { Div = 0, Axpy = 1 } kind = Div;
  int vec_sym = -1;                  // V
  struct Entry { int64_t e; int sum_sym, count_sym; };   // Axpy: sum_sym = g, count_sym = -1
  std::vector<Entry> entries;        // in program order
  std::vector<int> stmts;            // every statement of the group (temporaries and updates)
  Atom alpha;                        // Axpy
};

// A run of adjacent host statement pairs  a = VectorApply(X, e1);  VectorUpdate(V, e2, a)  (a read
// nowhere else) — the k-means centroid initialisation `mu.update(e, x.at(e))` of the staged
// programs.  Executed as device-to-device copies (contiguous segments coalesced) instead of
// 2 * len host statements that would each wait for the device.
struct CopyRun {
  int x_sym = -1, v_sym = -1;
  std::vector<std::pair<int64_t, int64_t>> pairs;   // (e1, e2) in program order
  std::vector<int> stmts;                           // every statement of the run
};

struct LoopPlan;   // a cached lowering (program.cpp)

struct Program {
  int root = -1;
  int max_sym = -1;
  int fused_pairs = 0;               // loop pairs fused by the executor ("fusion": "executor")
  std::vector<Stmt> stmts;           // indexed by sym; op == Unknown and sym == -1 for holes
  std::vector<Block> blocks;         // indexed by block id
  std::vector<uint8_t> has_block;
  // analyses
  std::vector<int32_t> uses;         // references to each sym (args, results, ranges, zeros)
  std::vector<uint8_t> print_only;   // every use of the sym is a Print argument
  std::unordered_map<int, UpdateGroup> update_after;   // loop stmt sym -> its update group
  std::unordered_map<int, CopyRun> copy_runs;          // first statement of the run -> run
  // lowering cache (loop stmt sym -> plan), filled by executions of this program
  mutable std::mutex plan_mu;
  mutable std::unordered_map<int, std::shared_ptr<LoopPlan>> plans;
  // per-symbol environments of finished executions, reused by the next ones (sizing and
  // clearing a max_sym-long environment per run is ~ms for a 10-iteration C4 program)
  mutable std::mutex scratch_mu;
  mutable std::vector<std::shared_ptr<void>> scratch;

  const Stmt& stmt(int s) const {
    if (s < 0 || s > max_sym || stmts[s].sym < 0) throw Fail(DLX_ERR_ARG, "malformed descriptor: no statement x" + std::to_string(s));
    return stmts[s];
  }
  const Block& block(int b) const {
    if (b < 0 || b >= static_cast<int>(blocks.size()) || !has_block[b])
      throw Fail(DLX_ERR_ARG, "malformed descriptor: no block " + std::to_string(b));
    return blocks[b];
  }
};

// Parses and analyses a dlx-program/1 descriptor (throws Fail / nlohmann exceptions).
std::shared_ptr<Program> parse_program(const char* text, size_t len);

std::string format_double(double x);

}  // namespace dlx
