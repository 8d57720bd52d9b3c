/*
 * oracle.h — CPU ORACLE for the fused-multiloop hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The product path (paper_1109_0778_b200/) never links,
 * loads or calls anything under oracle/.
 *
 * What it restates (the reference ships no interpreter or executor:
 * proj/include/stagekit/interp.hpp:10 is a declaration only, and executeDEG exists only
 * as prose in SPEC.md:645-663):
 *   - the per-index loop body / guarded left-fold order that emit_parallel_loop renders
 *     (proj/src/codegen.cpp:345-433): slots initialised to `zero`, one pass over
 *     i = 0..range-1, per elem `if (cond) acc = combine(acc, elem(i))`;
 *   - filtered-out indices contribute the identity (proj/include/stagekit/loops.hpp:22-24);
 *   - int64 wraparound (proj/src/graph.cpp:10-21) and IEEE fp64 without contraction
 *     (compiled with -ffp-contract=off, MiniC has separate * and +);
 *   - the Rng LCG (proj/include/stagekit/runtime.hpp:86-96), plus an O(log n)
 *     skip-ahead that is bit-identical to drawing sequentially;
 *   - SPEC.md:645-658 executeDEG: `chunks` contiguous index ranges, each folded
 *     sequentially from the elem's zero, partial activation records combined in
 *     ascending chunk order; chunks == 1 is the sequential interpreter.
 *   - format_double (proj/src/expr.cpp:11-22) for canonical result text.
 *
 * Pinned against SURVEY.md Appendix B known-answer values (JSON fixtures under tests/golden/), which
 * were derived by executing the reference's own emitted MiniC (see tests/golden/README.md).
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- Rng (runtime.hpp:86-96) ------------------------------------------------------ */
/* State after `n` next_unit() calls starting from `state` (affine LCG jump). */
uint64_t orc_rng_advance(uint64_t state, uint64_t n);
/* out[t] = the (first_draw + t)-th next_unit() of Rng(seed) (0-based draw numbering). */
void orc_rng_units(uint64_t seed, uint64_t first_draw, int64_t n, double* out, int threads);
/* out[t] = the (first_draw + t)-th next_int(bound) of Rng(seed). */
void orc_rng_ints(uint64_t seed, uint64_t first_draw, int64_t n, int64_t bound, int64_t* out,
                  int threads);

/* ---- k-means iteration (fused collect + k*(d+1) predicated reduces) ---------------- */
/* assign[i] = argmin_c sum_j (x[i*d+j]-mu[c*d+j])^2, chain `if (dist < best)` from
 * best = 1e300, index 0 (strict <, lowest index wins ties, NaN never wins);
 * counts[c] = #{i : assign[i]==c}, sums[c*d+j] = sum_{i: assign[i]==c} x[i*d+j].
 * workers/chunks: executeDEG parameters (chunks=1 -> sequential interpret). */
int orc_kmeans_step(const double* x, int64_t n, int32_t d, int32_t k, const double* mu,
                    int64_t* assign, int64_t* counts, double* sums, int workers, int chunks);
/* mu[c*d+j] = sums[c*d+j] / (double)counts[c]  (0/0 -> NaN, no trap: SPEC.md:670) */
void orc_kmeans_update(const int64_t* counts, const double* sums, int32_t k, int32_t d,
                       double* mu);

/* ---- GroupBy / bucket counts (K predicated count reduces `key(i)==b`) ------------- */
int orc_groupby_count(const int64_t* keys, int64_t n, int64_t nbuckets, int64_t* counts,
                      int workers, int chunks);

/* ---- Logistic regression gradient (fused dot -> sigmoid -> d reduces) ------------- */
/* h_i = 1/(1+exp(-(sum_j theta_j x_ij))), grad_j = sum_i (h_i - y_i) * x_ij.
 * exp is a documented extension: the reference op set has no exp (node.hpp:15-27). */
int orc_logreg_grad(const double* x, const int64_t* y, int64_t n, int32_t d,
                    const double* theta, double* grad, int workers, int chunks);

/* ---- GDA ---------------------------------------------------------------------------- */
/* pass 1: n1 = #{y==1}; sum0/sum1[j] = sum over class of x_ij  (1 + 2d predicated reduces) */
int orc_gda_pass1(const double* x, const int64_t* y, int64_t n, int32_t d, int64_t* n1,
                  double* sum0, double* sum1, int workers, int chunks);
/* pass 2: S[a*d+b] = sum_i (x_ia - mu_{y_i,a}) * (x_ib - mu_{y_i,b}), mu_y = y==1 ? mu1 : mu0 */
int orc_gda_pass2(const double* x, const int64_t* y, int64_t n, int32_t d, const double* mu0,
                  const double* mu1, double* scatter, int workers, int chunks);

/* ---- generic Map / ZipWith / Reduce families ---------------------------------------- */
/* out[i] = a * x[i] + y[i]  (axpy collect) */
void orc_axpy(double a, const double* x, const double* y, int64_t n, double* out);
/* sum_i x[i] (fp64 reduce, + combine) */
double orc_sum_f64(const double* x, int64_t n, int workers, int chunks);
/* sum_i x[i] (int64 reduce, wraparound) */
int64_t orc_sum_i64(const int64_t* x, int64_t n, int workers, int chunks);
/* mean + variance fused loop: sum and sum of squares (mean_variance demo) */
void orc_sum_sumsq_f64(const double* x, int64_t n, double* sum, double* sumsq, int workers,
                       int chunks);
/* count_where(x[i] > thr)  (count_gt7 demo family) */
int64_t orc_count_gt_f64(const double* x, int64_t n, double thr, int workers, int chunks);

/* ---- utilities ------------------------------------------------------------------------ */
uint64_t orc_fnv64w(const int64_t* v, int64_t n);
/* format_double (expr.cpp:11-22); returns length written (buf >= 64 bytes). */
int orc_format_double(double x, char* buf);
int orc_num_threads(void);

#ifdef __cplusplus
}
#endif
