// oracle.cpp — CPU ORACLE (test infrastructure only; see oracle.h for the contract and
// for what each function restates from the reference).  Compiled with
// -O3 -ffp-contract=off so that every fp64 `a*b + c` rounds twice, as the reference's
// MiniC `acc = acc + diff * diff` does.
#include "oracle.h"

#include <algorithm>
#include <atomic>
#include <charconv>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace {

constexpr uint64_t kMul = 6364136223846793005ULL;   // runtime.hpp:90
constexpr uint64_t kInc = 1442695040888963407ULL;   // runtime.hpp:90

inline double unit_of(uint64_t state) {              // runtime.hpp:91
  return static_cast<double>(state >> 11) * 0x1.0p-53;
}

// SPEC.md:645-658 executeDEG: split [0,n) into `chunks` contiguous ranges, run each
// chunk's process() sequentially on a pool of `workers` threads.  Chunk c covers
// [n*c/chunks, n*(c+1)/chunks).  The caller combines per-chunk activation records in
// ascending chunk order, so results never depend on `workers`.
template <class F>
void for_chunks(int64_t n, int workers, int chunks, F&& fn) {
  if (chunks < 1) chunks = 1;
  if (workers < 1) workers = 1;
  auto lo_of = [&](int c) { return static_cast<int64_t>((__int128)n * c / chunks); };
  if (workers == 1 || chunks == 1) {
    for (int c = 0; c < chunks; ++c) fn(c, lo_of(c), lo_of(c + 1));
    return;
  }
  std::atomic<int> next{0};
  std::vector<std::thread> pool;
  int nw = std::min(workers, chunks);
  pool.reserve(nw);
  for (int w = 0; w < nw; ++w)
    pool.emplace_back([&] {
      for (int c = next.fetch_add(1); c < chunks; c = next.fetch_add(1))
        fn(c, lo_of(c), lo_of(c + 1));
    });
  for (auto& t : pool) t.join();
}

inline int64_t wrap_add(int64_t a, int64_t b) {      // graph.cpp:10-13
  return static_cast<int64_t>(static_cast<uint64_t>(a) + static_cast<uint64_t>(b));
}

}  // namespace

extern "C" {

uint64_t orc_rng_advance(uint64_t state, uint64_t n) {
  // s_{t+1} = a*s_t + c.  Compose the affine map (A, C) = (a, c)^n by squaring.
  uint64_t acc_mul = 1, acc_add = 0, cur_mul = kMul, cur_add = kInc;
  while (n) {
    if (n & 1) {
      acc_mul = acc_mul * cur_mul;
      acc_add = acc_add * cur_mul + cur_add;
    }
    cur_add = (cur_mul + 1) * cur_add;
    cur_mul = cur_mul * cur_mul;
    n >>= 1;
  }
  return acc_mul * state + acc_add;
}

void orc_rng_units(uint64_t seed, uint64_t first_draw, int64_t n, double* out, int threads) {
  int chunks = std::max(1, threads) * 4;
  for_chunks(n, threads, chunks, [&](int, int64_t lo, int64_t hi) {
    uint64_t s = orc_rng_advance(seed, first_draw + static_cast<uint64_t>(lo));
    for (int64_t t = lo; t < hi; ++t) {
      s = s * kMul + kInc;
      out[t] = unit_of(s);
    }
  });
}

void orc_rng_ints(uint64_t seed, uint64_t first_draw, int64_t n, int64_t bound, int64_t* out,
                  int threads) {
  int chunks = std::max(1, threads) * 4;
  const double b = static_cast<double>(bound);
  for_chunks(n, threads, chunks, [&](int, int64_t lo, int64_t hi) {
    uint64_t s = orc_rng_advance(seed, first_draw + static_cast<uint64_t>(lo));
    for (int64_t t = lo; t < hi; ++t) {
      s = s * kMul + kInc;
      out[t] = static_cast<int64_t>(unit_of(s) * b);   // runtime.hpp:93-95
    }
  });
}

int orc_kmeans_step(const double* x, int64_t n, int32_t d, int32_t k, const double* mu,
                    int64_t* assign, int64_t* counts, double* sums, int workers, int chunks) {
  if (n < 0 || d <= 0 || k <= 0) return 1;
  if (chunks < 1) chunks = 1;
  // mu transposed (d x k) so the per-centroid accumulators vectorise across c while each
  // accumulator is still the sequential j-order chain acc = acc + diff*diff.
  std::vector<double> mut(static_cast<size_t>(d) * k);
  for (int c = 0; c < k; ++c)
    for (int j = 0; j < d; ++j) mut[static_cast<size_t>(j) * k + c] = mu[static_cast<size_t>(c) * d + j];
  std::vector<int64_t> pc(static_cast<size_t>(chunks) * k, 0);
  std::vector<double> ps(static_cast<size_t>(chunks) * k * d, 0.0);
  for_chunks(n, workers, chunks, [&](int ch, int64_t lo, int64_t hi) {
    std::vector<double> acc(k);
    int64_t* cc = &pc[static_cast<size_t>(ch) * k];
    double* cs = &ps[static_cast<size_t>(ch) * k * d];
    for (int64_t i = lo; i < hi; ++i) {
      const double* xi = x + i * d;
      for (int c = 0; c < k; ++c) acc[c] = 0.0;
      for (int j = 0; j < d; ++j) {
        const double xj = xi[j];
        const double* mj = &mut[static_cast<size_t>(j) * k];
        for (int c = 0; c < k; ++c) {
          const double diff = xj - mj[c];
          acc[c] = acc[c] + diff * diff;
        }
      }
      double best = 1e300;   // argmin chain initial value (staged_if chain, stage.cpp:73-104)
      int64_t bi = 0;
      for (int c = 0; c < k; ++c)
        if (acc[c] < best) { best = acc[c]; bi = c; }
      assign[i] = bi;
      cc[bi] = wrap_add(cc[bi], 1);
      double* srow = cs + bi * d;
      for (int j = 0; j < d; ++j) srow[j] = srow[j] + xi[j];
    }
  });
  // ascending-chunk combine of the activation records
  for (int c = 0; c < k; ++c) counts[c] = 0;
  for (int64_t t = 0; t < static_cast<int64_t>(k) * d; ++t) sums[t] = 0.0;
  for (int ch = 0; ch < chunks; ++ch) {
    for (int c = 0; c < k; ++c) counts[c] = wrap_add(counts[c], pc[static_cast<size_t>(ch) * k + c]);
    const double* cs = &ps[static_cast<size_t>(ch) * k * d];
    if (ch == 0) {
      for (int64_t t = 0; t < static_cast<int64_t>(k) * d; ++t) sums[t] = cs[t];
    } else {
      for (int64_t t = 0; t < static_cast<int64_t>(k) * d; ++t) sums[t] = sums[t] + cs[t];
    }
  }
  return 0;
}

void orc_kmeans_update(const int64_t* counts, const double* sums, int32_t k, int32_t d,
                       double* mu) {
  for (int c = 0; c < k; ++c) {
    const double cnt = static_cast<double>(counts[c]);   // toDouble
    for (int j = 0; j < d; ++j) mu[c * d + j] = sums[c * d + j] / cnt;
  }
}

int orc_groupby_count(const int64_t* keys, int64_t n, int64_t nbuckets, int64_t* counts,
                      int workers, int chunks) {
  if (nbuckets <= 0) return 1;
  if (chunks < 1) chunks = 1;
  std::vector<int64_t> pc(static_cast<size_t>(chunks) * nbuckets, 0);
  for_chunks(n, workers, chunks, [&](int ch, int64_t lo, int64_t hi) {
    int64_t* cc = &pc[static_cast<size_t>(ch) * nbuckets];
    for (int64_t i = lo; i < hi; ++i) {
      const int64_t key = keys[i];
      // K predicated reduces `if (key(i) == b) cnt_b = cnt_b + 1`: keys outside
      // [0, K) match no guard and contribute nothing.
      if (key >= 0 && key < nbuckets) cc[key] = wrap_add(cc[key], 1);
    }
  });
  for (int64_t b = 0; b < nbuckets; ++b) counts[b] = 0;
  for (int ch = 0; ch < chunks; ++ch)
    for (int64_t b = 0; b < nbuckets; ++b)
      counts[b] = wrap_add(counts[b], pc[static_cast<size_t>(ch) * nbuckets + b]);
  return 0;
}

int orc_logreg_grad(const double* x, const int64_t* y, int64_t n, int32_t d,
                    const double* theta, double* grad, int workers, int chunks) {
  if (d <= 0) return 1;
  if (chunks < 1) chunks = 1;
  std::vector<double> pg(static_cast<size_t>(chunks) * d, 0.0);
  for_chunks(n, workers, chunks, [&](int ch, int64_t lo, int64_t hi) {
    double* g = &pg[static_cast<size_t>(ch) * d];
    for (int64_t i = lo; i < hi; ++i) {
      const double* xi = x + i * d;
      double z = 0.0;
      for (int j = 0; j < d; ++j) z = z + theta[j] * xi[j];
      const double h = 1.0 / (1.0 + std::exp(-z));
      const double r = h - static_cast<double>(y[i]);
      for (int j = 0; j < d; ++j) g[j] = g[j] + r * xi[j];
    }
  });
  for (int j = 0; j < d; ++j) grad[j] = pg[j];
  for (int ch = 1; ch < chunks; ++ch)
    for (int j = 0; j < d; ++j) grad[j] = grad[j] + pg[static_cast<size_t>(ch) * d + j];
  return 0;
}

int orc_gda_pass1(const double* x, const int64_t* y, int64_t n, int32_t d, int64_t* n1,
                  double* sum0, double* sum1, int workers, int chunks) {
  if (d <= 0) return 1;
  if (chunks < 1) chunks = 1;
  std::vector<int64_t> pn(chunks, 0);
  std::vector<double> p0(static_cast<size_t>(chunks) * d, 0.0), p1(static_cast<size_t>(chunks) * d, 0.0);
  for_chunks(n, workers, chunks, [&](int ch, int64_t lo, int64_t hi) {
    double* s0 = &p0[static_cast<size_t>(ch) * d];
    double* s1 = &p1[static_cast<size_t>(ch) * d];
    int64_t cnt = 0;
    for (int64_t i = lo; i < hi; ++i) {
      const double* xi = x + i * d;
      if (y[i] == 1) {
        cnt = wrap_add(cnt, 1);
        for (int j = 0; j < d; ++j) s1[j] = s1[j] + xi[j];
      }
      if (y[i] == 0) {
        for (int j = 0; j < d; ++j) s0[j] = s0[j] + xi[j];
      }
    }
    pn[ch] = cnt;
  });
  *n1 = 0;
  for (int ch = 0; ch < chunks; ++ch) *n1 = wrap_add(*n1, pn[ch]);
  for (int j = 0; j < d; ++j) { sum0[j] = p0[j]; sum1[j] = p1[j]; }
  for (int ch = 1; ch < chunks; ++ch)
    for (int j = 0; j < d; ++j) {
      sum0[j] = sum0[j] + p0[static_cast<size_t>(ch) * d + j];
      sum1[j] = sum1[j] + p1[static_cast<size_t>(ch) * d + j];
    }
  return 0;
}

int orc_gda_pass2(const double* x, const int64_t* y, int64_t n, int32_t d, const double* mu0,
                  const double* mu1, double* scatter, int workers, int chunks) {
  if (d <= 0) return 1;
  if (chunks < 1) chunks = 1;
  const size_t dd = static_cast<size_t>(d) * d;
  std::vector<double> ps(static_cast<size_t>(chunks) * dd, 0.0);
  for_chunks(n, workers, chunks, [&](int ch, int64_t lo, int64_t hi) {
    double* s = &ps[static_cast<size_t>(ch) * dd];
    std::vector<double> diff(d);
    for (int64_t i = lo; i < hi; ++i) {
      const double* xi = x + i * d;
      const double* m = (y[i] == 1) ? mu1 : mu0;   // per-element IfThenElse select
      for (int j = 0; j < d; ++j) diff[j] = xi[j] - m[j];
      for (int a = 0; a < d; ++a) {
        const double da = diff[a];
        double* row = s + static_cast<size_t>(a) * d;
        for (int b = 0; b < d; ++b) row[b] = row[b] + da * diff[b];
      }
    }
  });
  for (size_t t = 0; t < dd; ++t) scatter[t] = ps[t];
  for (int ch = 1; ch < chunks; ++ch)
    for (size_t t = 0; t < dd; ++t) scatter[t] = scatter[t] + ps[static_cast<size_t>(ch) * dd + t];
  return 0;
}

void orc_axpy(double a, const double* x, const double* y, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = a * x[i] + y[i];
}

double orc_sum_f64(const double* x, int64_t n, int workers, int chunks) {
  if (chunks < 1) chunks = 1;
  std::vector<double> p(chunks, 0.0);
  for_chunks(n, workers, chunks, [&](int ch, int64_t lo, int64_t hi) {
    double acc = 0.0;
    for (int64_t i = lo; i < hi; ++i) acc = acc + x[i];
    p[ch] = acc;
  });
  double r = p[0];
  for (int ch = 1; ch < chunks; ++ch) r = r + p[ch];
  return r;
}

int64_t orc_sum_i64(const int64_t* x, int64_t n, int workers, int chunks) {
  if (chunks < 1) chunks = 1;
  std::vector<int64_t> p(chunks, 0);
  for_chunks(n, workers, chunks, [&](int ch, int64_t lo, int64_t hi) {
    int64_t acc = 0;
    for (int64_t i = lo; i < hi; ++i) acc = wrap_add(acc, x[i]);
    p[ch] = acc;
  });
  int64_t r = 0;
  for (int ch = 0; ch < chunks; ++ch) r = wrap_add(r, p[ch]);
  return r;
}

void orc_sum_sumsq_f64(const double* x, int64_t n, double* sum, double* sumsq, int workers,
                       int chunks) {
  if (chunks < 1) chunks = 1;
  std::vector<double> p(chunks, 0.0), q(chunks, 0.0);
  for_chunks(n, workers, chunks, [&](int ch, int64_t lo, int64_t hi) {
    double a = 0.0, b = 0.0;
    for (int64_t i = lo; i < hi; ++i) {
      a = a + x[i];
      b = b + x[i] * x[i];
    }
    p[ch] = a;
    q[ch] = b;
  });
  double a = p[0], b = q[0];
  for (int ch = 1; ch < chunks; ++ch) { a = a + p[ch]; b = b + q[ch]; }
  *sum = a;
  *sumsq = b;
}

int64_t orc_count_gt_f64(const double* x, int64_t n, double thr, int workers, int chunks) {
  if (chunks < 1) chunks = 1;
  std::vector<int64_t> p(chunks, 0);
  for_chunks(n, workers, chunks, [&](int ch, int64_t lo, int64_t hi) {
    int64_t acc = 0;
    for (int64_t i = lo; i < hi; ++i)
      if (thr < x[i]) acc = wrap_add(acc, 1);
    p[ch] = acc;
  });
  int64_t r = 0;
  for (int ch = 0; ch < chunks; ++ch) r = wrap_add(r, p[ch]);
  return r;
}

uint64_t orc_fnv64w(const int64_t* v, int64_t n) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (int64_t i = 0; i < n; ++i) {
    h ^= static_cast<uint64_t>(v[i]);
    h *= 0x100000001b3ULL;
  }
  return h;
}

int orc_format_double(double x, char* buf) {
  std::string s;
  if (std::isnan(x)) {
    s = "nan";
  } else if (std::isinf(x)) {
    s = x > 0 ? "inf" : "-inf";
  } else {
    char tmp[64];
    auto res = std::to_chars(tmp, tmp + sizeof(tmp), x);
    s.assign(tmp, res.ptr);
    if (s.find('.') == std::string::npos && s.find('e') == std::string::npos) s += ".0";
  }
  std::memcpy(buf, s.data(), s.size());
  buf[s.size()] = '\0';
  return static_cast<int>(s.size());
}

int orc_num_threads(void) {
  unsigned h = std::thread::hardware_concurrency();
  return h ? static_cast<int>(h) : 1;
}

}  // extern "C"
