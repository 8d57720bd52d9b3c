"""Pin the CPU oracle against the reference-derived known answers (SPEC.md
examples).  CPU only."""
import hashlib

import numpy as np
import pytest

import oracle as O


def test_rng_kats(golden):
    r = golden["rng"]
    assert O.rng_units(1, 0, 4).tolist() == r["seed1_units"]
    assert O.rng_ints(1, 0, 8, 64).tolist() == r["seed1_ints64"]
    assert O.rng_units(42, 0, 4).tolist() == r["seed42_units"]
    assert O.rng_ints(42, 0, 8, 64).tolist() == r["seed42_ints64"]
    assert hex(O.rng_advance(1, 2 ** 20)) == r["seed1_state_after_2p20"]
    assert hex(O.rng_advance(1, 10 ** 9)) == r["seed1_state_after_1e9"]


def test_rng_skip_ahead_matches_sequential():
    seq = O.rng_units(7, 0, 10_000, nthreads=1)
    for start in (0, 1, 999, 4097):
        assert np.array_equal(O.rng_units(7, start, 1000, nthreads=4), seq[start:start + 1000])
    ints = O.rng_ints(7, 0, 5000, 1000, nthreads=1)
    assert np.array_equal(O.rng_ints(7, 123, 77, 1000, nthreads=3), ints[123:200])


def test_c1_kmeans_goldens(golden):
    g = golden["c1_kmeans"]
    x, mu0 = O.kmeans_inputs(g["n"], g["d"], g["k"], g["seed"])
    hist = O.kmeans_run(x, g["k"], g["iters"], mu0)
    for it, (counts, _, mu, _, _) in enumerate(hist):
        assert counts.tolist() == g["counts"][it], f"iteration {it + 1}"
        assert O.format_double(mu[0, 0]) == g["mu00"][it]
    counts, _, mu, _, _ = hist[-1]
    text = O.kmeans_canonical_text(counts, mu)
    assert hashlib.sha256(text.encode()).hexdigest() == g["final_text_sha256"]
    assert [O.format_double(v) for v in mu[0, :4]] == g["final_mu_row0_prefix"]


def test_c1_assignment_hashes(oracle_hashes):
    x, mu0 = O.kmeans_inputs(65536, 16, 8)
    hist = O.kmeans_run(x, 8, 10, mu0)
    assert [hex(h[1]) for h in hist] == oracle_hashes["c1_assign_fnv64w"]


@pytest.mark.parametrize("workers,chunks", [(1, 1), (2, 8), (8, 32), (3, 7)])
def test_kmeans_chunking_assignments_independent(workers, chunks):
    """executeDEG contract: assignments/counts do not depend on chunking; fp sums within 1e-9."""
    x, mu0 = O.kmeans_inputs(20000, 16, 8, seed=3)
    a1, c1, s1 = O.kmeans_step(x, 8, mu0)
    a2, c2, s2 = O.kmeans_step(x, 8, mu0, workers=workers, chunks=chunks)
    assert np.array_equal(a1, a2) and np.array_equal(c1, c2)
    np.testing.assert_allclose(s2, s1, rtol=1e-12)


def test_chunked_result_independent_of_workers():
    """Double reduce bit-identical for workers in {1, 8} at chunks = 64."""
    x = O.rng_units(5, 0, 1_000_003)
    assert O.sum_f64(x, workers=1, chunks=64) == O.sum_f64(x, workers=8, chunks=64)
    x2, mu0 = O.kmeans_inputs(30000, 16, 8, seed=9)
    r1 = O.kmeans_step(x2, 8, mu0, workers=1, chunks=64)
    r8 = O.kmeans_step(x2, 8, mu0, workers=8, chunks=64)
    for a, b in zip(r1, r8):
        assert np.array_equal(a, b)


def test_spec_examples():
    ints = np.arange(1, 10 ** 6 + 1, dtype=np.int64)
    for w in (1, 2, 8):
        assert O.sum_i64(ints, workers=w, chunks=max(4 * w, 1)) == 500000500000
    const = np.full(1000, 0.3)
    s, sq = O.sum_sumsq_f64(const)
    mean = s / 1000
    assert abs(sq / 1000 - mean * mean) < 1e-12
    x = O.rng_units(11, 0, 1000)
    s, sq = O.sum_sumsq_f64(x)
    np.testing.assert_allclose(s / 1000, x.mean(), rtol=1e-9)
    np.testing.assert_allclose(sq / 1000 - (s / 1000) ** 2, x.var(), rtol=1e-9)
    y = O.rng_units(12, 0, 1000)
    assert np.array_equal(O.axpy(2.5, x, y), 2.5 * x + y)
    assert O.count_gt_f64(x * 10, 7.0) == int(np.sum(x * 10 > 7.0))


def test_int_wraparound():
    v = np.array([2 ** 62, 2 ** 62, 2 ** 62], dtype=np.int64)
    assert O.sum_i64(v) == -(2 ** 62)  # graph.cpp:10-21 two's-complement wrap


def test_kmeans_edge_semantics():
    # ties -> lowest index; NaN centroid never wins; all-NaN -> index 0 (chain start)
    x = np.array([[0.0, 0.0], [1.0, 1.0], [0.5, 0.5]])
    mu = np.array([[1.0, 1.0], [1.0, 1.0], [0.0, 0.0]])
    a, c, s = O.kmeans_step(x, 3, mu)
    assert a.tolist() == [2, 0, 0]
    mu_nan = np.array([[np.nan, np.nan], [1.0, 1.0]])
    a, _, _ = O.kmeans_step(x, 2, mu_nan)
    assert a.tolist() == [1, 1, 1]
    a, c, _ = O.kmeans_step(x, 2, np.full((2, 2), np.nan))
    assert a.tolist() == [0, 0, 0] and c.tolist() == [3, 0]
    # empty cluster -> 0/0 = NaN centroid (no trap)
    mu2 = O.kmeans_update(np.array([3, 0]), np.array([[1.0, 2.0], [0.0, 0.0]]))
    assert np.isnan(mu2[1]).all()


def test_groupby_out_of_range_keys():
    keys = np.array([0, 1, 1, -1, 5, 4, 2, 1 << 40], dtype=np.int64)
    assert O.groupby_count(keys, 5).tolist() == [1, 2, 1, 0, 1]


def test_c3_gda_goldens(golden):
    g = golden["c3_gda"]
    n, d = g["n"], g["d"]
    x = O.rng_units(1, 0, n * d).reshape(n, d)
    y = O.rng_ints(1, n * d, n, 2)
    n1, s0, s1 = O.gda_pass1(x, y)
    assert n1 == g["n1"]
    mu0, mu1 = s0 / float(n - n1), s1 / float(n1)
    S = O.gda_pass2(x, y, mu0, mu1)
    assert O.format_double(mu0[0]) == g["mu0_0"] and O.format_double(mu1[0]) == g["mu1_0"]
    assert O.format_double(S[0, 0]) == g["S00"] and O.format_double(S[0, 1]) == g["S01"]
    assert O.format_double(S[63, 63]) == g["S6363"]
    text = O.gda_canonical_text(n1, mu0, mu1, S)
    assert hashlib.sha256(text.encode()).hexdigest() == g["text_sha256"]


@pytest.mark.slow
def test_c4_kmeans_first_iteration(golden, oracle_hashes):
    g = golden["c4_kmeans"]
    x, mu0 = O.kmeans_inputs(g["n"], g["d"], g["k"], g["seed"])
    a, c, s = O.kmeans_step(x, g["k"], mu0, workers=O.threads(), chunks=4 * O.threads())
    assert c[:4].tolist() == g["counts_prefix"][0]
    assert hex(O.fnv64w(a)) == oracle_hashes["c4_assign_fnv64w"][0]
    np.testing.assert_allclose(s[0, 0], float(g["sum_c0_d0"][0]), rtol=1e-12)


@pytest.mark.slow
@pytest.mark.parametrize("K", ["64", "4096", "65536"])
def test_c5_groupby_goldens(golden, oracle_hashes, K):
    g = golden["c5_groupby"]["by_k"][K]
    keys = O.rng_ints(1, 0, golden["c5_groupby"]["n"], int(K))
    c = O.groupby_count(keys, int(K), workers=O.threads(), chunks=4 * O.threads())
    assert [c[0], c[-1], c.min(), c.max()] == [g["first"], g["last"], g["min"], g["max"]]
    assert hex(O.fnv64w(c)) == oracle_hashes["c5_counts_fnv64w"][K]


def test_logreg_oracle_matches_numpy():
    n, d = 3000, 16
    x = O.rng_units(2, 0, n * d).reshape(n, d)
    y = O.rng_ints(2, n * d, n, 2)
    th = np.linspace(-1, 1, d)
    g = O.logreg_grad(x, y, th)
    h = 1.0 / (1.0 + np.exp(-(x @ th)))
    np.testing.assert_allclose(g, (h - y) @ x, rtol=1e-10)
    assert np.array_equal(O.logreg_grad(x, y, th, workers=4, chunks=16), O.logreg_grad(x, y, th, workers=1, chunks=16))
