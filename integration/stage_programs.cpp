// stage_programs.cpp — stages the hot-path programs through the reference DSL (stagekit,
// built out of tree by oracle/ref.mk), fuses them with the reference's own fuse_loops (code
// motion off: SURVEY §0.3), schedules, runs the reference's run_codegen, and writes for each
// program one fixture JSON under tests/golden/staged/:
//   - "program":  the executor descriptor (integration/stagekit_dlx.cpp::to_dlx_program)
//   - "deg":      the reference's DEG JSON (codegen.cpp:569-588)
//   - "minic":    the reference's emitted MiniC text
//   - "expected": the output text of that MiniC program, executed by the oracle's MiniC
//                 evaluator (oracle/minic_eval.hpp, the restated missing interp.cpp)
// The GPU tests run "program" through dlx_program_run and compare with "expected".
//
//   oracle/_ref/stage_programs OUT_DIR [NAME]  (built by `make -C oracle -f ref.mk`)
// With NAME only that program is staged; the headline-shape programs
// "kmeans_n16777216_d64_k64_it1[_unfused]" (C4, k*(d+1) = 4,160 reduces) are staged only on
// request and write only the descriptor (OUT/NAME.program.json; the sequential MiniC evaluation
// of 16M x 64 x 64 would take hours): the fused one takes the reference's quadratic fuse_loops
// (> 25 min), the unfused one ~6 s and is fused by the executor (csrc/fuse.cpp).
// Programs named *_unfused skip fuse_loops and are serialised with "fusion": "executor".
#include <chrono>
#include <cstdio>
#include <fstream>
#include <functional>
#include <iostream>
#include <json.hpp>
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
using json = nlohmann::ordered_json;

namespace {

DVal plus(Stage& st, DVal a, DVal b) { return DVal{&st, st.numeric(Op::Plus, a.e, b.e)}; }

// k-means: one collect (argmin chain over k inner distance reduces) + k*(d+1) predicated
// reduces per iteration; mu is a mutable vector updated from sums/counts; the assignment
// vector escapes (printed) so fusion keeps its elem live.  With all_assign every
// iteration prints the whole assignment vector (not only row 0), so the GPU's assignments are
// pinned element by element to what the reference's own emitted program computes.
void kmeans(Stage& st, int64_t n, int d, int k, int iters, bool all_assign = false) {
  DVec x = vec_rand(st, st.lit(n * d));
  DVec mu = vec_alloc(st, st.lit(int64_t{k} * d), SemType::f64());
  for (int e = 0; e < k * d; ++e) mu.update(st.lit(int64_t{e}), x.at(st.lit(int64_t{e})));
  for (int it = 0; it < iters; ++it) {
    DVec assign = mk_collect(st, st.lit(n), [&](DInt i) -> DVal {
      DDouble best = st.lit(1e300);
      DInt idx = st.lit(int64_t{0});
      for (int c = 0; c < k; ++c) {
        DDouble dist(mk_reduce(
            st, st.lit(int64_t{d}), st.lit(0.0),
            [&](DInt j) -> DVal {
              DDouble xv = x.at_d(i * st.lit(int64_t{d}) + j);
              DDouble mv = mu.at_d(st.lit(int64_t{c} * d) + j);
              DDouble diff = xv - mv;
              return diff * diff;
            },
            [&](DVal l, DVal r) { return plus(st, l, r); }));
        DBool lt = dist < best;
        best = st.if_then_else<DDouble>(lt, [&] { return dist; }, [&] { return best; });
        idx = st.if_then_else<DInt>(lt, [&] { return st.lit(int64_t{c}); }, [&] { return idx; });
      }
      return idx;
    });
    for (int64_t r = 0; r < (all_assign ? n : 1); ++r) st.print(assign.at_i(st.lit(r)));
    std::vector<DInt> counts;
    std::vector<DDouble> sums;
    for (int c = 0; c < k; ++c) {
      std::function<DBool(DInt)> in_c = [&, c](DInt i) { return assign.at_i(i) == st.lit(int64_t{c}); };
      counts.push_back(DInt(mk_reduce(
          st, st.lit(n), st.lit(int64_t{0}), [&](DInt) -> DVal { return st.lit(int64_t{1}); },
          [&](DVal l, DVal r) { return plus(st, l, r); }, &in_c)));
      for (int j = 0; j < d; ++j)
        sums.push_back(DDouble(mk_reduce(
            st, st.lit(n), st.lit(0.0),
            [&, j](DInt i) -> DVal { return x.at(i * st.lit(int64_t{d}) + st.lit(int64_t{j})); },
            [&](DVal l, DVal r) { return plus(st, l, r); }, &in_c)));
    }
    for (int c = 0; c < k; ++c) {
      st.print(counts[c]);
      DDouble cnt = st.to_double(counts[c]);
      for (int j = 0; j < d; ++j) mu.update(st.lit(int64_t{c} * d + j), sums[c * d + j] / cnt);
    }
  }
  for (int e = 0; e < k * d; ++e) st.print(mu.at(st.lit(int64_t{e})));
}

// GroupBy / Naive-Bayes counts: K predicated count reduces keyed on a random int vector.
void groupby(Stage& st, int64_t n, int K) {
  DVec keys = vec_rand_int(st, st.lit(n), st.lit(int64_t{K}));
  std::vector<DInt> cnt;
  for (int b = 0; b < K; ++b) {
    std::function<DBool(DInt)> is_b = [&, b](DInt i) { return keys.at_i(i) == st.lit(int64_t{b}); };
    cnt.push_back(DInt(mk_reduce(
        st, st.lit(n), st.lit(int64_t{0}), [&](DInt) -> DVal { return st.lit(int64_t{1}); },
        [&](DVal l, DVal r) { return plus(st, l, r); }, &is_b)));
  }
  for (auto& c : cnt) st.print(c);
}

// GDA: pass 1 (class count + per-class sums), pass 2 (d*d scatter with per-class mean select).
void gda(Stage& st, int64_t n, int d) {
  DVec x = vec_rand(st, st.lit(n * d));
  DVec y = vec_rand_int(st, st.lit(n), st.lit(int64_t{2}));
  std::function<DBool(DInt)> is1 = [&](DInt i) { return y.at_i(i) == st.lit(int64_t{1}); };
  std::function<DBool(DInt)> is0 = [&](DInt i) { return y.at_i(i) == st.lit(int64_t{0}); };
  DInt n1(mk_reduce(st, st.lit(n), st.lit(int64_t{0}), [&](DInt) -> DVal { return st.lit(int64_t{1}); },
                    [&](DVal l, DVal r) { return plus(st, l, r); }, &is1));
  std::vector<DDouble> mu0, mu1;
  DDouble nn1 = st.to_double(n1);
  DDouble nn0 = st.to_double(st.lit(n) - n1);
  for (int j = 0; j < d; ++j) {
    auto xj = [&, j](DInt i) -> DVal { return x.at(i * st.lit(int64_t{d}) + st.lit(int64_t{j})); };
    DDouble s0(mk_reduce(st, st.lit(n), st.lit(0.0), xj, [&](DVal l, DVal r) { return plus(st, l, r); }, &is0));
    DDouble s1(mk_reduce(st, st.lit(n), st.lit(0.0), xj, [&](DVal l, DVal r) { return plus(st, l, r); }, &is1));
    mu0.push_back(s0 / nn0);
    mu1.push_back(s1 / nn1);
  }
  st.print(n1);
  for (int j = 0; j < d; ++j) {
    st.print(mu0[j]);
    st.print(mu1[j]);
  }
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b) {
      DDouble s(mk_reduce(
          st, st.lit(n), st.lit(0.0),
          [&, a, b](DInt i) -> DVal {
            DBool c1 = y.at_i(i) == st.lit(int64_t{1});
            DDouble ma = st.if_then_else<DDouble>(c1, [&] { return mu1[a]; }, [&] { return mu0[a]; });
            DDouble mb = st.if_then_else<DDouble>(c1, [&] { return mu1[b]; }, [&] { return mu0[b]; });
            DDouble da = x.at_d(i * st.lit(int64_t{d}) + st.lit(int64_t{a})) - ma;
            DDouble db = x.at_d(i * st.lit(int64_t{d}) + st.lit(int64_t{b})) - mb;
            return da * db;
          },
          [&](DVal l, DVal r) { return plus(st, l, r); }));
      st.print(s);
    }
}

// Logistic regression BGD in the collect form: h = link(theta . x_i) escapes
// (printed), so fusion keeps one loop of 1 collect + d gradient reduces
// (h(i) - y(i)) * x(i*d + j); then theta(j) -= alpha * g_j on the host.  The reference op set
// has no exp (node.hpp:15-27), so the link is the softsign stand-in t / (1 + |t|) the survey
// staged; the executor's logistic family evaluates whatever link expression the loop carries.
void logreg(Stage& st, int64_t n, int d, int iters, double alpha) {
  DVec x = vec_rand(st, st.lit(n * d));
  DVec y = vec_rand_int(st, st.lit(n), st.lit(int64_t{2}));
  DVec th = vec_alloc(st, st.lit(int64_t{d}), SemType::f64());
  for (int it = 0; it < iters; ++it) {
    DVec h = mk_collect(st, st.lit(n), [&](DInt i) -> DVal {
      DDouble dot(mk_reduce(
          st, st.lit(int64_t{d}), st.lit(0.0),
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
      th.update(st.lit(int64_t{j}), th.at_d(st.lit(int64_t{j})) - st.lit(alpha) * g[j]);
  }
  for (int j = 0; j < d; ++j) st.print(th.at(st.lit(int64_t{j})));
}

// mean_variance demo: mean and variance fuse into one loop.
void mean_variance(Stage& st, int64_t n) {
  DVec x = vec_rand(st, st.lit(n));
  st.print(mean(st, x));
  st.print(variance(st, x));
}

// axpy demo: a*x + y collect, then a sum and two element reads.
void axpy(Stage& st, int64_t n) {
  DVec x = vec_rand(st, st.lit(n));
  DVec y = vec_rand(st, st.lit(n));
  DDouble a = st.lit(2.5);
  DVec z = x.zip_with(y, [&](DVal u, DVal v) -> DVal { return a * DDouble(u) + DDouble(v); });
  st.print(z.at(st.lit(int64_t{0})));
  st.print(z.at(st.lit(n - 1)));
  st.print(z.sum());
}

// count_gt7 demo family: a predicated count over a scaled random vector.
void count_gt(Stage& st, int64_t n) {
  DVec x = vec_rand(st, st.lit(n));
  st.print(x.count_where([&](DVal v) { return st.lit(0.7) < DDouble(v); }));
  st.print(x.sum());
}

// SPADE-style find + count: a filter-collect (find_indexes, an append
// collect: loops.cpp:105-109, vectordsl.cpp:153-160) fused with a predicated count over the
// same range, then reads of the appended vector (its length, first element, and a sum loop
// over it).
void find_count(Stage& st, int64_t n) {
  DVec x = vec_rand(st, st.lit(n));
  DVec hits = x.find_indexes([&](DVal v) { return st.lit(0.9) < DDouble(v); });
  st.print(x.count_where([&](DVal v) { return st.lit(0.9) < DDouble(v); }));
  st.print(hits.len());
  st.print(hits.at(st.lit(int64_t{0})));
  st.print(hits.sum());
}

// Fusion-legality probes (the executor's fusion pass must refuse these pairs, as the
// reference's fuse_loops does): a sum over a mutable vector, an update of it, and the same sum
// again (the second loop reads a vector written between the two); a sum, a map that subtracts
// it (reads the first loop's reduce result) and the map's sum; a map over x and a sum over a
// vector of another length (different ranges).
void fusion_blockers(Stage& st, int64_t n) {
  DVec m = vec_alloc(st, st.lit(int64_t{8}), SemType::f64());
  for (int e = 0; e < 8; ++e) m.update(st.lit(int64_t{e}), st.lit(0.5 * e));
  st.print(m.sum());
  m.update(st.lit(int64_t{3}), st.lit(100.0));
  st.print(m.sum());
  DVec x = vec_rand(st, st.lit(n));
  DDouble s(x.sum());
  DVec y = x.map([&](DVal v) -> DVal { return DDouble(v) - s; });
  st.print(y.sum());
  DVec z = vec_rand(st, st.lit(n / 2));
  st.print(z.sum());
  st.print(y.at(st.lit(int64_t{1})));
}

struct Spec {
  std::string name;
  std::function<void(Stage&)> body;
};

}  // namespace

int main(int argc, char** argv) {
  const std::string out_dir = argc > 1 ? argv[1] : "tests/golden/staged";
  const uint64_t seed = 1;
  std::vector<Spec> specs = {
      {"kmeans_n4096_d16_k8_it2", [](Stage& st) { kmeans(st, 4096, 16, 8, 2); }},
      {"kmeans_n65536_d16_k8_it1", [](Stage& st) { kmeans(st, 65536, 16, 8, 1); }},
      {"kmeans_n4096_d16_k8_it2_assign", [](Stage& st) { kmeans(st, 4096, 16, 8, 2, true); }},
      {"groupby_n100000_k16", [](Stage& st) { groupby(st, 100000, 16); }},
      {"gda_n20000_d4", [](Stage& st) { gda(st, 20000, 4); }},
      {"logreg_n20000_d8_it2", [](Stage& st) { logreg(st, 20000, 8, 2, 1.0 / 20000); }},
      {"mean_variance_n100000", [](Stage& st) { mean_variance(st, 100000); }},
      {"axpy_n100000", [](Stage& st) { axpy(st, 100000); }},
      {"count_gt_n100000", [](Stage& st) { count_gt(st, 100000); }},
      {"find_count_n100000", [](Stage& st) { find_count(st, 100000); }},
      // unfused: the reference's fuse_loops is skipped and the executor fuses the root loops
      // (csrc/fuse.cpp); "expected" is the unfused program's own MiniC output (it equals the
      // fused program's)
      {"kmeans_n4096_d16_k8_it2_unfused", [](Stage& st) { kmeans(st, 4096, 16, 8, 2); }},
      {"groupby_n100000_k16_unfused", [](Stage& st) { groupby(st, 100000, 16); }},
      {"gda_n20000_d4_unfused", [](Stage& st) { gda(st, 20000, 4); }},
      {"logreg_n20000_d8_it2_unfused", [](Stage& st) { logreg(st, 20000, 8, 2, 1.0 / 20000); }},
      {"mean_variance_n100000_unfused", [](Stage& st) { mean_variance(st, 100000); }},
      {"find_count_n100000_unfused", [](Stage& st) { find_count(st, 100000); }},
      {"axpy_n100000_unfused", [](Stage& st) { axpy(st, 100000); }},
      {"count_gt_n100000_unfused", [](Stage& st) { count_gt(st, 100000); }},
      {"fusion_blockers_n10000", [](Stage& st) { fusion_blockers(st, 10000); }},
      {"gda_n20000_d16", [](Stage& st) { gda(st, 20000, 16); }},
      {"gda_n20000_d16_unfused", [](Stage& st) { gda(st, 20000, 16); }},
      {"logreg_n20000_d16_it3", [](Stage& st) { logreg(st, 20000, 16, 3, 1.0 / 20000); }},
      {"logreg_n20000_d16_it3_unfused", [](Stage& st) { logreg(st, 20000, 16, 3, 1.0 / 20000); }},
      // the headline shape (d = k = 64) at a small N: the reference's fuse_loops cannot fuse it
      // in reasonable time, so only the unfused program exists; its MiniC output is evaluated
      {"kmeans_n4096_d64_k64_it2_unfused", [](Stage& st) { kmeans(st, 4096, 64, 64, 2); }},
      {"fusion_blockers_n10000_unfused", [](Stage& st) { fusion_blockers(st, 10000); }},
  };
  const std::string only = argc > 2 ? argv[2] : "";
  if (only == "kmeans_n16777216_d64_k64_it1" || only == "kmeans_n16777216_d64_k64_it1_unfused")
    specs = {{only, [](Stage& st) { kmeans(st, 16777216, 64, 64, 1); }}};
  const bool eval = only.rfind("kmeans_n16777216", 0) != 0;
  auto ends_with = [](const std::string& a, const std::string& b) {
    return a.size() >= b.size() && a.compare(a.size() - b.size(), b.size(), b) == 0;
  };
  for (const Spec& sp : specs) {
    if (!only.empty() && sp.name != only) continue;
    const auto t0 = std::chrono::steady_clock::now();
    Stage st;
    st.begin();
    sp.body(st);
    st.finish();
    auto g = st.take_graph();
    const bool unfused = ends_with(sp.name, "_unfused");
    FusionOutcome fo;
    if (unfused) fo.graph = g;
    else fo = fuse_loops(g, /*with_motion=*/false);
    Schedule s = build_schedule(*fo.graph, ScheduleOptions{true, false});
    const auto t1 = std::chrono::steady_clock::now();
    const std::string program = unfused ? stagekit_dlx::to_dlx_program_unfused(*fo.graph, s)
                                        : stagekit_dlx::to_dlx_program(*fo.graph, s);
    const auto t1s = std::chrono::steady_clock::now();
    if (!eval) {   // production shape: the descriptor alone (no MiniC: codegen renders 4,161 loops)
      std::ofstream(out_dir + "/" + sp.name + ".program.json") << program << "\n";
      std::printf("%-28s stage+schedule %.2fs  serialise %.2fs  %zu bytes\n", sp.name.c_str(),
                  std::chrono::duration<double>(t1 - t0).count(),
                  std::chrono::duration<double>(t1s - t1).count(), program.size());
      continue;
    }
    CodegenResult cg = run_codegen(*fo.graph, s);
    oracle_minic::Evaluator ev(seed);
    oracle_minic::EvalResult r;
    if (eval) r = ev.run(cg.program);
    const auto t2 = std::chrono::steady_clock::now();
    int loops = 0;
    for (int32_t idx : s.block_stmts(fo.graph->root()))
      if (fo.graph->stmts()[idx].is_loop()) ++loops;
    json fx;
    fx["name"] = sp.name;
    fx["seed"] = seed;
    fx["fused_pairs"] = fo.fused_pairs;
    fx["root_loops"] = loops;
    fx["program"] = json::parse(program);
    fx["deg"] = unfused ? json(nullptr) : json::parse(cg.deg_json);
    if (sp.name.size() > 7 && sp.name.compare(sp.name.size() - 7, 7, "_assign") == 0) {
      // the DEG's ordered-effect anti-dependence lists grow quadratically with the 8,192 Print
      // statements (322 MB); the executor never reads it, so this fixture carries none
      fx["program"].erase("deg");
      fx["deg"] = nullptr;
    }
    fx["minic"] = cg.minic_text;
    if (eval) fx["expected"] = r.output;
    std::ofstream(out_dir + "/" + sp.name + ".json") << fx.dump(1) << "\n";
    std::printf("%-28s fused_pairs=%d root_loops=%d stage+fuse+codegen %.2fs  minic eval %.2fs\n",
                sp.name.c_str(), fo.fused_pairs, loops,
                std::chrono::duration<double>(t1 - t0).count(),
                std::chrono::duration<double>(t2 - t1).count());
  }
  return 0;
}
