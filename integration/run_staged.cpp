// run_staged.cpp — end-to-end drop-in check in C++: stage programs with the REFERENCE DSL
// (stagekit, built out of tree by oracle/ref.mk), fuse + schedule them with the reference's
// own passes, then execute them twice — with the reference's emitted MiniC on the CPU
// (oracle/minic_eval.hpp, the restated interpret()) and on the B200 through
// stagekit_dlx::run_on_b200 (the C ABI) — and compare the printed outputs (Int exact, Double
// rtol 1e-9).  Exit code 0 iff every program matches.  Run on a GPU box:
//   oracle/_ref/run_staged
#include <cmath>
#include <cstdio>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

#include "integration/stagekit_dlx.hpp"
#include "oracle/minic_eval.hpp"
#include "stagekit/codegen.hpp"
#include "stagekit/fusion.hpp"
#include "stagekit/loops.hpp"
#include "stagekit/stage.hpp"
#include "stagekit/vectordsl.hpp"

using namespace stagekit;

namespace {

DVal plus(Stage& st, DVal a, DVal b) { return DVal{&st, st.numeric(Op::Plus, a.e, b.e)}; }

void kmeans(Stage& st, int64_t n, int d, int k) {
  DVec x = vec_rand(st, st.lit(n * d));
  DVec assign = mk_collect(st, st.lit(n), [&](DInt i) -> DVal {
    DDouble best = st.lit(1e300);
    DInt idx = st.lit(int64_t{0});
    for (int c = 0; c < k; ++c) {
      DDouble dist(mk_reduce(
          st, st.lit(int64_t{d}), st.lit(0.0),
          [&](DInt j) -> DVal {
            DDouble diff = x.at_d(i * st.lit(int64_t{d}) + j) - x.at_d(st.lit(int64_t{c} * d) + j);
            return diff * diff;
          },
          [&](DVal l, DVal r) { return plus(st, l, r); }));
      DBool lt = dist < best;
      best = st.if_then_else<DDouble>(lt, [&] { return dist; }, [&] { return best; });
      idx = st.if_then_else<DInt>(lt, [&] { return st.lit(int64_t{c}); }, [&] { return idx; });
    }
    return idx;
  });
  st.print(assign.at_i(st.lit(int64_t{0})));
  for (int c = 0; c < k; ++c) {
    std::function<DBool(DInt)> in_c = [&, c](DInt i) { return assign.at_i(i) == st.lit(int64_t{c}); };
    st.print(DInt(mk_reduce(st, st.lit(n), st.lit(int64_t{0}), [&](DInt) -> DVal { return st.lit(int64_t{1}); },
                            [&](DVal l, DVal r) { return plus(st, l, r); }, &in_c)));
    for (int j = 0; j < d; ++j)
      st.print(DDouble(mk_reduce(
          st, st.lit(n), st.lit(0.0),
          [&, j](DInt i) -> DVal { return x.at(i * st.lit(int64_t{d}) + st.lit(int64_t{j})); },
          [&](DVal l, DVal r) { return plus(st, l, r); }, &in_c)));
  }
}

void stats(Stage& st, int64_t n) {
  DVec x = vec_rand(st, st.lit(n));
  st.print(mean(st, x));
  st.print(variance(st, x));
  st.print(x.count_where([&](DVal v) { return st.lit(0.5) < DDouble(v); }));
  DVec keys = vec_rand_int(st, st.lit(n), st.lit(int64_t{8}));
  for (int b = 0; b < 8; ++b) st.print(keys.count_where([&, b](DVal v) { return DInt(v) == st.lit(int64_t{b}); }));
}

// the C3 / C2 shapes at small size: GDA (pass 1 keyed sums + pass 2 scatter) and logistic
// regression in the collect form with the softsign link (the reference has no exp)
void gda(Stage& st, int64_t n, int d) {
  DVec x = vec_rand(st, st.lit(n * d));
  DVec y = vec_rand_int(st, st.lit(n), st.lit(int64_t{2}));
  std::function<DBool(DInt)> is1 = [&](DInt i) { return y.at_i(i) == st.lit(int64_t{1}); };
  std::function<DBool(DInt)> is0 = [&](DInt i) { return y.at_i(i) == st.lit(int64_t{0}); };
  DInt n1(mk_reduce(st, st.lit(n), st.lit(int64_t{0}), [&](DInt) -> DVal { return st.lit(int64_t{1}); },
                    [&](DVal l, DVal r) { return plus(st, l, r); }, &is1));
  std::vector<DDouble> mu0, mu1;
  DDouble nn1 = st.to_double(n1), nn0 = st.to_double(st.lit(n) - n1);
  for (int j = 0; j < d; ++j) {
    auto xj = [&, j](DInt i) -> DVal { return x.at(i * st.lit(int64_t{d}) + st.lit(int64_t{j})); };
    mu0.push_back(DDouble(mk_reduce(st, st.lit(n), st.lit(0.0), xj, [&](DVal l, DVal r) { return plus(st, l, r); }, &is0)) / nn0);
    mu1.push_back(DDouble(mk_reduce(st, st.lit(n), st.lit(0.0), xj, [&](DVal l, DVal r) { return plus(st, l, r); }, &is1)) / nn1);
  }
  st.print(n1);
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b)
      st.print(DDouble(mk_reduce(
          st, st.lit(n), st.lit(0.0),
          [&, a, b](DInt i) -> DVal {
            DBool c1 = y.at_i(i) == st.lit(int64_t{1});
            DDouble ma = st.if_then_else<DDouble>(c1, [&] { return mu1[a]; }, [&] { return mu0[a]; });
            DDouble mb = st.if_then_else<DDouble>(c1, [&] { return mu1[b]; }, [&] { return mu0[b]; });
            return (x.at_d(i * st.lit(int64_t{d}) + st.lit(int64_t{a})) - ma) *
                   (x.at_d(i * st.lit(int64_t{d}) + st.lit(int64_t{b})) - mb);
          },
          [&](DVal l, DVal r) { return plus(st, l, r); })));
}

void logreg(Stage& st, int64_t n, int d, int iters) {
  DVec x = vec_rand(st, st.lit(n * d));
  DVec y = vec_rand_int(st, st.lit(n), st.lit(int64_t{2}));
  DVec th = vec_alloc(st, st.lit(int64_t{d}), SemType::f64());
  for (int it = 0; it < iters; ++it) {
    DVec h = mk_collect(st, st.lit(n), [&](DInt i) -> DVal {
      DDouble dot(mk_reduce(st, st.lit(int64_t{d}), st.lit(0.0),
                            [&](DInt j) -> DVal { return th.at_d(j) * x.at_d(i * st.lit(int64_t{d}) + j); },
                            [&](DVal l, DVal r) { return plus(st, l, r); }));
      return dot / (st.lit(1.0) + DDouble(st.abs(dot)));
    });
    st.print(h.at(st.lit(int64_t{0})));
    std::vector<DDouble> g;
    for (int j = 0; j < d; ++j)
      g.push_back(DDouble(mk_reduce(
          st, st.lit(n), st.lit(0.0),
          [&, j](DInt i) -> DVal {
            return (h.at_d(i) - st.to_double(y.at_i(i))) * x.at_d(i * st.lit(int64_t{d}) + st.lit(int64_t{j}));
          },
          [&](DVal l, DVal r) { return plus(st, l, r); })));
    for (int j = 0; j < d; ++j)
      th.update(st.lit(int64_t{j}), th.at_d(st.lit(int64_t{j})) - st.lit(1.0 / static_cast<double>(n)) * g[j]);
  }
  for (int j = 0; j < d; ++j) st.print(th.at(st.lit(int64_t{j})));
}

bool same(const std::string& a, const std::string& b) {
  if (a == b) return true;
  try {
    const double x = std::stod(a), y = std::stod(b);
    if (a.find('.') == std::string::npos && a.find('e') == std::string::npos) return false;  // ints exact
    return std::fabs(x - y) <= 1e-9 * std::max(std::fabs(x), std::fabs(y));
  } catch (...) {
    return false;
  }
}

}  // namespace

int main() {
  struct Case {
    const char* name;
    std::function<void(Stage&)> body;
  };
  std::vector<Case> cases = {{"kmeans_n65536_d16_k8", [](Stage& st) { kmeans(st, 65536, 16, 8); }},
                             {"stats_groupby_n1000000", [](Stage& st) { stats(st, 1000000); }},
                             {"gda_n50000_d16", [](Stage& st) { gda(st, 50000, 16); }},
                             {"logreg_n100000_d16_it3", [](Stage& st) { logreg(st, 100000, 16, 3); }}};
  int failures = 0;
  for (const Case& cs : cases) {
    Stage st;
    st.begin();
    cs.body(st);
    st.finish();
    auto g = st.take_graph();
    FusionOutcome fo = fuse_loops(g, false);
    Schedule s = build_schedule(*fo.graph, ScheduleOptions{true, false});
    CodegenResult cg = run_codegen(*fo.graph, s);
    oracle_minic::Evaluator ev(1);
    const std::string ref = ev.run(cg.program).output;
    RunResult got;
    try {
      got = stagekit_dlx::run_on_b200(*fo.graph, s, 1, 0);
    } catch (const std::exception& e) {
      std::printf("%s: B200 run failed: %s\n", cs.name, e.what());
      ++failures;
      continue;
    }
    std::istringstream a(ref), b(got.output);
    std::string la, lb;
    int lines = 0, bad = 0;
    while (std::getline(a, la)) {
      if (!std::getline(b, lb) || !same(la, lb)) ++bad;
      ++lines;
    }
    if (std::getline(b, lb)) ++bad;
    std::printf("%-26s fused_pairs=%d lines=%d mismatches=%d -> %s\n", cs.name, fo.fused_pairs, lines, bad,
                bad ? "FAIL" : "PASS");
    failures += bad != 0;
  }
  return failures ? 1 : 0;
}
