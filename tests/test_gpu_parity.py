"""GPU parity: every CUDA family against the CPU oracle on the same seeded inputs, through the
C ABI.  Bit-exact for integer / index results (assignments, counts, GroupBy); rtol 1e-9 for
fp64 sums (north-star tolerance; the reduction order differs from the sequential fold)."""
import hashlib
import zlib

import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RTOL = 1e-9  # fp64 sums (north_star: "1e-9 fp64")
SCREENED = 2  # dlx_kmeans_step method: tcgen05 screen + exact recheck


@pytest.fixture(scope="module")
def ml():
    assert torch.cuda.is_available()
    from paper_1109_0778_b200 import multiloops
    return multiloops


def dev_units(ml, n, d, seed=1, first=0):
    return ml.rng_units(n * d, seed=seed, first_draw=first).view(n, d)


# ---- Rng ------------------------------------------------------------------------------------

@pytest.mark.parametrize("n,seed,first", [(1, 1, 0), (1000, 1, 0), (123457, 42, 99), (3_000_001, 7, 10 ** 9)])
def test_rng_bit_identical(ml, n, seed, first):
    assert np.array_equal(ml.rng_units(n, seed=seed, first_draw=first).cpu().numpy(), O.rng_units(seed, first, n))
    for b in (2, 64, 65536):
        assert np.array_equal(ml.rng_ints(n, b, seed=seed, first_draw=first).cpu().numpy(),
                              O.rng_ints(seed, first, n, b))


# ---- k-means ----------------------------------------------------------------------------------

def check_step(ml, x, mu, method=0):
    xh, muh = x.cpu().numpy(), mu.cpu().numpy()
    a, c, s = ml.kmeans_step(x, mu, method=method)
    a_ref, c_ref, s_ref = O.kmeans_step(np.ascontiguousarray(xh), mu.shape[0], muh)
    assert np.array_equal(a.cpu().numpy().astype(np.int64), a_ref)
    assert np.array_equal(c.cpu().numpy(), c_ref)
    np.testing.assert_allclose(s.cpu().numpy(), s_ref, rtol=RTOL, atol=0)
    return a_ref, c_ref, s_ref


@pytest.mark.parametrize("method", [0, 1, SCREENED])
def test_c1_stepwise_ten_iterations(ml, golden, method):
    """at every iteration run the GPU step from the oracle's centroids."""
    g = golden["c1_kmeans"]
    x = dev_units(ml, g["n"], g["d"])
    mu = x[: g["k"]].clone()
    for it in range(g["iters"]):
        _, c_ref, s_ref = check_step(ml, x, mu, method)
        assert c_ref.tolist() == g["counts"][it]
        mu = torch.from_numpy(O.kmeans_update(c_ref, s_ref)).cuda()


def test_c1_free_running(ml, golden):
    from paper_1109_0778_b200.programs import KMeansProgram
    g = golden["c1_kmeans"]
    x = dev_units(ml, g["n"], g["d"])
    prog = KMeansProgram(x, g["k"], x[: g["k"]])
    for it in range(g["iters"]):
        prog.step()
        assert prog.counts.cpu().tolist() == g["counts"][it]
    mu = prog.mu.cpu().numpy()
    assert O.format_double(mu[0, 0]) == g["mu00"][-1] or abs(mu[0, 0] - float(g["mu00"][-1])) < 1e-12
    text = O.kmeans_canonical_text(prog.counts.cpu().numpy(), mu)
    print("C1 GPU free-running text sha256:", hashlib.sha256(text.encode()).hexdigest())


def test_kmeans_graph_equals_eager(ml):
    from paper_1109_0778_b200.programs import KMeansProgram
    x = dev_units(ml, 50_000, 32, seed=5)
    e = KMeansProgram(x, 16, x[:16]).run(4)
    gph = KMeansProgram(x, 16, x[:16]).capture().run(4)
    assert torch.equal(e.mu, gph.mu) and torch.equal(e.counts, gph.counts)


@pytest.mark.parametrize("n,d,k", [(1, 16, 8), (37, 5, 3), (1000, 64, 64), (5000, 33, 17), (3000, 130, 10),
                                   (2048, 16, 1), (4099, 64, 64), (10_000, 2, 70), (777, 96, 24),
                                   (1_000_003, 16, 8), (300_001, 64, 8), (200_000, 7, 64)])
@pytest.mark.parametrize("method", [0, 1])
def test_kmeans_shapes(ml, n, d, k, method):
    x = dev_units(ml, n, d, seed=n + d + k)
    mu = dev_units(ml, k, d, seed=99)
    check_step(ml, x, mu, method)



@pytest.mark.parametrize("n,d,k", [(1, 16, 8), (1000, 64, 64), (4099, 64, 64), (2048, 16, 1), (300_001, 64, 64),
                                   (70_000, 2, 3), (5000, 40, 33), (129, 64, 64), (100_000, 32, 16)])
def test_kmeans_screened_shapes(ml, n, d, k):
    x = dev_units(ml, n, d, seed=n + 7 * d + k)
    mu = dev_units(ml, k, d, seed=5)
    check_step(ml, x, mu, SCREENED)


@pytest.mark.parametrize("n,k", [(128, 64), (255, 64), (128 * 148 + 1, 64), (40_000, 32), (40_000, 1)])
def test_kmeans_screened_tile_edges(ml, n, k):
    """d = 64 tile edges: exactly one tile, a shifted last tile overlapping its predecessor,
    one row past a full wave of CTAs, and fewer centroids than one N half."""
    x = dev_units(ml, n, 64, seed=n + k)
    mu = dev_units(ml, k, 64, seed=11)
    check_step(ml, x, mu, SCREENED)


def test_kmeans_screened_unaligned_rows(ml):
    """Rows starting 16 bytes past a 32-byte boundary take the 16-byte-load variant."""
    n, d, k = 30_001, 64, 64
    base = dev_units(ml, n * d + 2, 1, seed=3).view(-1)
    x = base[2:].view(n, d)
    assert x.data_ptr() % 32 == 16
    check_step(ml, x, dev_units(ml, k, d, seed=4), SCREENED)


def _stress_inputs(kind, n=20_000, d=64, k=64):
    g = torch.Generator(device="cpu").manual_seed(zlib.crc32(kind.encode()))
    x = torch.rand(n, d, generator=g, dtype=torch.float64)
    mu = x[torch.randperm(n, generator=g)[:k]].clone()
    if kind == "signed":
        x = 2 * x - 1
        mu = 2 * mu - 1
    elif kind == "scaled_rows":
        x = x * torch.pow(10.0, torch.randint(-3, 4, (n, 1), generator=g).double())
    elif kind == "integer_ties":
        x = torch.floor(x * 4)
        mu = torch.floor(mu * 4)
    elif kind == "dup_centroids":
        mu[1::2] = mu[0::2]
    elif kind == "points_on_centroids":
        x[: 2 * k] = mu.repeat(2, 1)
    elif kind == "nonfinite_rows":
        x[5, 3] = float("nan")
        x[777, 0] = float("inf")
        x[12345, 63] = -float("inf")
    elif kind == "nonfinite_centroids":
        mu[3] = float("nan")
        mu[9, 5] = float("inf")
    elif kind == "huge":
        x = x * 1e200
        mu = mu * 1e200
    elif kind == "tiny":
        x = x * 1e-300
        mu = mu * 1e-300
    elif kind == "zeros":
        x = torch.zeros_like(x)
        mu = torch.zeros_like(mu)
    elif kind == "centroids_far":
        mu = mu * 1e3
    elif kind == "samples_far":
        x = x * 1e4
    return x.cuda(), mu.cuda()


@pytest.mark.parametrize("kind", ["signed", "scaled_rows", "integer_ties", "dup_centroids", "points_on_centroids",
                                  "nonfinite_rows", "nonfinite_centroids", "huge", "tiny", "zeros", "centroids_far",
                                  "samples_far"])
@pytest.mark.parametrize("method", [0, SCREENED])
def test_kmeans_screened_stress(ml, kind, method):
    x, mu = _stress_inputs(kind)
    xh, muh = x.cpu().numpy(), mu.cpu().numpy()
    a, c, s = ml.kmeans_step(x, mu, method=method)
    a_ref, c_ref, s_ref = O.kmeans_step(np.ascontiguousarray(xh), mu.shape[0], muh)
    assert np.array_equal(a.cpu().numpy().astype(np.int64), a_ref)
    assert np.array_equal(c.cpu().numpy(), c_ref)
    np.testing.assert_allclose(s.cpu().numpy(), s_ref, rtol=RTOL, atol=0, equal_nan=True)


def test_kmeans_screened_recheck_fraction(ml):
    x = dev_units(ml, 1 << 20, 64, seed=1)
    ml.kmeans_step(x, x[:64].clone(), method=SCREENED)
    r = ml.kmeans_last_recheck_count(1 << 20, 64, 64)
    print(f"screened recheck fraction at N=2^20, d=k=64: {r / (1 << 20):.5f}")
    assert 0 <= r < (1 << 20) // 10


def test_screened_rejects_unsupported(ml):
    from paper_1109_0778_b200 import GenerationFailed
    x = dev_units(ml, 100, 65, seed=1)
    with pytest.raises(GenerationFailed):
        ml.kmeans_step(x, x[:4].clone(), method=SCREENED)
    x = dev_units(ml, 100, 16, seed=1)
    with pytest.raises(GenerationFailed):
        ml.kmeans_step(x, dev_units(ml, 65, 16), method=SCREENED)


def test_kmeans_ties_and_nan(ml):
    x = dev_units(ml, 4000, 16, seed=3)
    mu = x[:8].clone()
    mu[5] = mu[2]          # duplicate centroid: lower index must win every tie
    mu[7] = float("nan")   # empty-cluster centroid: never wins
    check_step(ml, x, mu)
    check_step(ml, x, torch.full_like(mu, float("nan")))   # all NaN -> chain start index 0
    xi = torch.zeros(64, 4, dtype=torch.float64, device="cuda")
    check_step(ml, xi, torch.zeros(3, 4, dtype=torch.float64, device="cuda"))  # exact ties


def test_kmeans_empty_cluster_update(ml):
    counts = torch.tensor([3, 0], dtype=torch.int64, device="cuda")
    sums = torch.tensor([[1.0, 2.0], [0.0, 0.0]], dtype=torch.float64, device="cuda")
    mu = ml.kmeans_update(counts, sums).cpu().numpy()
    assert np.isnan(mu[1]).all() and mu[0].tolist() == [1.0 / 3.0, 2.0 / 3.0]


@pytest.mark.parametrize("method", [0, 1])
def test_c4_first_two_iterations(ml, golden, oracle_hashes, method):
    g = golden["c4_kmeans"]
    x = dev_units(ml, g["n"], g["d"])
    mu = x[: g["k"]].clone()
    xh = x.cpu().numpy()
    for it in range(2):
        a, c, s = ml.kmeans_step(x, mu, method=method)
        a_h = a.cpu().numpy().astype(np.int64)
        assert hex(O.fnv64w(a_h)) == oracle_hashes["c4_assign_fnv64w"][it]
        assert c.cpu().tolist()[:4] == g["counts_prefix"][it]
        sums = s.cpu().numpy()
        np.testing.assert_allclose(sums[0, 0], float(g["sum_c0_d0"][it]), rtol=RTOL)
        # the oracle's sums for the same assignments (chunked; rtol) drive the next step
        _, c_ref, s_ref = O.kmeans_step(xh, g["k"], mu.cpu().numpy(), workers=O.threads(), chunks=4 * O.threads())
        np.testing.assert_allclose(sums, s_ref, rtol=RTOL)
        mu = torch.from_numpy(O.kmeans_update(c_ref, s_ref)).cuda()


def test_c4_free_running_ten_iterations(ml, golden):
    """the GPU and the oracle each run C4's 10 iterations on their OWN centroids (no
    re-seeding from the oracle); the number of assignments that differ per iteration is 0 and
    the counts agree exactly, so the fp64 sum-order differences (rtol 1e-9) never flip a
    nearest-centroid decision at this workload."""
    g = golden["c4_kmeans"]
    n, d, k = g["n"], g["d"], g["k"]
    x = dev_units(ml, n, d)
    xh = x.cpu().numpy()
    mu_g = x[:k].clone()
    mu_o = xh[:k].copy()
    diffs = []
    for it in range(10):
        a, c, s = ml.kmeans_step(x, mu_g)
        a_o, c_o, s_o = O.kmeans_step(xh, k, mu_o, workers=O.threads(), chunks=4 * O.threads())
        diffs.append(int(np.count_nonzero(a.cpu().numpy().astype(np.int64) != a_o)))
        assert c.cpu().numpy().tolist() == c_o.tolist(), (it, diffs)
        np.testing.assert_allclose(s.cpu().numpy(), s_o, rtol=RTOL)
        mu_g = ml.kmeans_update(c, s)
        mu_o = O.kmeans_update(c_o, s_o)
        np.testing.assert_allclose(mu_g.cpu().numpy(), mu_o, rtol=RTOL)
    assert diffs == [0] * 10


# ---- GroupBy ------------------------------------------------------------------------------------

@pytest.mark.parametrize("n,K", [(1, 64), (1001, 64), (1_000_003, 64), (1_000_000, 4096), (999_999, 65536),
                                 (77_777, 30_001), (1, 65536), (500_000, 200_000), (400_001, 300_001),
                                 (300_000, 500_000), (100, 1)])
def test_groupby(ml, n, K):
    keys = ml.rng_ints(n, K, seed=K)
    assert np.array_equal(ml.groupby_count(keys, K).cpu().numpy(), O.groupby_count(keys.cpu().numpy(), K))


def test_groupby_out_of_range(ml):
    keys = torch.tensor([0, 1, 1, -1, 5, 4, 2, 1 << 40, 3], dtype=torch.int64, device="cuda")
    assert ml.groupby_count(keys, 5).cpu().tolist() == [1, 2, 1, 1, 1]
    assert ml.groupby_count(keys, 300_000).cpu().numpy()[:6].tolist() == [1, 2, 1, 1, 1, 1]
    assert ml.groupby_count(keys, 50_001).cpu().numpy()[:6].tolist() == [1, 2, 1, 1, 1, 1]   # cluster path


@pytest.mark.parametrize("key", [0, 40_000, 65_535])
def test_groupby_cluster_one_hot_bucket(ml, key):
    """Every key in one bucket (local or partner-SM half of the two-CTA histogram): maximal
    contention on a single distributed-shared-memory counter."""
    n = 3_000_001
    keys = torch.full((n,), key, dtype=torch.int64, device="cuda")
    c = ml.groupby_count(keys, 65536).cpu().numpy()
    assert c[key] == n and c.sum() == n


@pytest.mark.parametrize("K", ["64", "4096", "65536"])
def test_c5_groupby(ml, golden, oracle_hashes, K):
    g = golden["c5_groupby"]["by_k"][K]
    keys = ml.rng_ints(golden["c5_groupby"]["n"], int(K), seed=1)
    c = ml.groupby_count(keys, int(K)).cpu().numpy()
    assert [c[0], c[-1], c.min(), c.max()] == [g["first"], g["last"], g["min"], g["max"]]
    assert hex(O.fnv64w(c)) == oracle_hashes["c5_counts_fnv64w"][K]
    del keys
    torch.cuda.empty_cache()


# ---- logistic regression --------------------------------------------------------------------------

@pytest.mark.parametrize("n,d", [(1, 64), (1000, 64), (1_048_576, 64), (3001, 2), (5000, 130), (4096, 256)])
def test_logreg_grad(ml, n, d):
    x = dev_units(ml, n, d, seed=4)
    y = ml.rng_ints(n, 2, seed=4, first_draw=n * d)
    th = torch.linspace(-0.3, 0.3, d, dtype=torch.float64, device="cuda")
    g = ml.logreg_grad(x, y, th).cpu().numpy()
    ref = O.logreg_grad(x.cpu().numpy(), y.cpu().numpy(), th.cpu().numpy(), workers=O.threads(), chunks=4 * O.threads())
    np.testing.assert_allclose(g, ref, rtol=RTOL, atol=1e-9 * np.abs(ref).max())


@pytest.mark.parametrize("n,d", [(1, 64), (1000, 64), (1_048_576, 64), (3001, 2), (5000, 130), (4096, 256)])
def test_logreg_grad_f32_storage(ml, n, d):
    """The fp32-storage opt-in (dlx_logreg_grad_f32): x held as float, promoted exactly; the
    gradient is bit-identical to the fp64 kernel on the promoted matrix and matches the oracle
    on it (rtol 1e-9)."""
    x32 = dev_units(ml, n, d, seed=5).float()
    xp = x32.double()
    y = ml.rng_ints(n, 2, seed=5, first_draw=n * d)
    th = torch.linspace(-0.3, 0.3, d, dtype=torch.float64, device="cuda")
    g32 = ml.logreg_grad(x32, y, th)
    g64 = ml.logreg_grad(xp, y, th)
    assert torch.equal(g32, g64)
    ref = O.logreg_grad(xp.cpu().numpy(), y.cpu().numpy(), th.cpu().numpy(), workers=O.threads(), chunks=4 * O.threads())
    np.testing.assert_allclose(g32.cpu().numpy(), ref, rtol=RTOL, atol=1e-9 * np.abs(ref).max())
    # against the reference on the ORIGINAL fp64 inputs: north_star's fp32 tolerance, 1e-5
    x64 = dev_units(ml, n, d, seed=5)
    ref64 = O.logreg_grad(x64.cpu().numpy(), y.cpu().numpy(), th.cpu().numpy(), workers=O.threads(), chunks=4 * O.threads())
    np.testing.assert_allclose(g32.cpu().numpy(), ref64, rtol=1e-5, atol=1e-5 * np.abs(ref64).max())


def test_logreg_bgd_f32_storage_program(ml):
    """BGD through LogRegProgram (CUDA-graph iterations) on fp32-stored x equals the fp64 program
    on the promoted matrix bit for bit."""
    from paper_1109_0778_b200.programs import LogRegProgram
    n, d, iters = 1_048_576, 64, 5
    x32 = dev_units(ml, n, d).float()
    y = ml.rng_ints(n, 2, seed=1, first_draw=n * d)
    a = LogRegProgram(x32, y, torch.zeros(d, dtype=torch.float64, device="cuda"), 1.0 / n).capture()
    b = LogRegProgram(x32.double(), y, torch.zeros(d, dtype=torch.float64, device="cuda"), 1.0 / n).capture()
    for _ in range(iters):
        a.step()
        b.step()
    assert torch.equal(a.theta, b.theta)


def test_c2_logreg_bgd_20_iterations(ml):
    from paper_1109_0778_b200.programs import LogRegProgram
    n, d, iters = 1_048_576, 64, 20
    alpha = 1.0 / n
    x = dev_units(ml, n, d)
    y = ml.rng_ints(n, 2, seed=1, first_draw=n * d)
    prog = LogRegProgram(x, y, torch.zeros(d, dtype=torch.float64, device="cuda"), alpha).capture()
    xh, yh = x.cpu().numpy(), y.cpu().numpy()
    th = np.zeros(d)
    for _ in range(iters):
        prog.step()
        th = th - alpha * O.logreg_grad(xh, yh, th, workers=O.threads(), chunks=4 * O.threads())
    np.testing.assert_allclose(prog.theta.cpu().numpy(), th, rtol=1e-9, atol=1e-13)


# ---- GDA ---------------------------------------------------------------------------------------------

def test_c3_gda(ml, golden):
    g = golden["c3_gda"]
    n, d = g["n"], g["d"]
    x = dev_units(ml, n, d)
    y = ml.rng_ints(n, 2, seed=1, first_draw=n * d)
    n1, mu0, mu1, S = ml.gda(x, y)
    assert int(n1.item()) == g["n1"]
    mu0, mu1, S = mu0.cpu().numpy(), mu1.cpu().numpy(), S.cpu().numpy()
    np.testing.assert_allclose(mu0[0], float(g["mu0_0"]), rtol=RTOL)
    np.testing.assert_allclose(mu1[0], float(g["mu1_0"]), rtol=RTOL)
    np.testing.assert_allclose([S[0, 0], S[0, 1], S[63, 63]], [float(g["S00"]), float(g["S01"]), float(g["S6363"])],
                               rtol=RTOL)
    xh, yh = x.cpu().numpy(), y.cpu().numpy()
    n1r, s0, s1 = O.gda_pass1(xh, yh, workers=O.threads(), chunks=4 * O.threads())
    m0, m1 = s0 / float(n - n1r), s1 / float(n1r)
    np.testing.assert_allclose(mu0, m0, rtol=RTOL)
    np.testing.assert_allclose(mu1, m1, rtol=RTOL)
    Sr = O.gda_pass2(xh, yh, m0, m1, workers=O.threads(), chunks=4 * O.threads())
    np.testing.assert_allclose(S, Sr, rtol=RTOL, atol=1e-9 * np.abs(Sr).max())


@pytest.mark.parametrize("n,d", [(1, 2), (999, 16), (5000, 30), (4097, 100), (2000, 128), (300_001, 64), (37_893, 48), (128 * 148 * 2 + 5, 64)])
def test_gda_shapes(ml, n, d):
    x = dev_units(ml, n, d, seed=8)
    y = ml.rng_ints(n, 2, seed=8, first_draw=n * d)
    n1, mu0, mu1, S = ml.gda(x, y)
    xh, yh = x.cpu().numpy(), y.cpu().numpy()
    n1r, s0, s1 = O.gda_pass1(xh, yh)
    assert int(n1.item()) == n1r
    with np.errstate(all="ignore"):
        m0, m1 = s0 / float(n - n1r), s1 / float(n1r)
    np.testing.assert_allclose(mu0.cpu().numpy(), m0, rtol=RTOL)
    np.testing.assert_allclose(mu1.cpu().numpy(), m1, rtol=RTOL)
    if np.isfinite(m0).all() and np.isfinite(m1).all():
        Sr = O.gda_pass2(xh, yh, m0, m1)
        np.testing.assert_allclose(S.cpu().numpy(), Sr, rtol=RTOL, atol=1e-9 * max(1.0, np.abs(Sr).max()))


def _gda_two_pass(ml, x, y):
    n1, s0, s1 = ml.gda_pass1(x, y)
    mu0, mu1 = ml.gda_means(n1, s0, s1, x.shape[0])
    return n1, mu0, mu1, ml.gda_pass2(x, y, mu0, mu1)


@pytest.mark.parametrize("n,d", [(1, 64), (63, 64), (64, 64), (65, 64), (10_000, 64), (1_048_576, 64), (5_001, 17), (40_000, 32)])
def test_gda_fit_matches_two_pass(ml, n, d):
    """The single-pass fit (shifted scatter + rank-1 correction) against the reference's two
    passes on the same device, and its certification flag stays clear on iid data."""
    x = dev_units(ml, n, d, seed=9)
    y = ml.rng_ints(n, 2, seed=9, first_draw=n * d)
    f = ml.gda_fit(x, y)
    assert not ml.gda_fit_last_fallback(x) or n < 2
    if d % 2:   # the two-pass row kernels need even d; the fit does not: check it on the oracle
        xh, yh = x.cpu().numpy(), y.cpu().numpy()
        n1r, s0, s1 = O.gda_pass1(xh, yh)
        m0, m1 = s0 / float(n - n1r), s1 / float(n1r)
        t = (torch.tensor([n1r]), torch.from_numpy(m0), torch.from_numpy(m1),
             torch.from_numpy(O.gda_pass2(xh, yh, m0, m1)))
    else:
        t = _gda_two_pass(ml, x, y)
    assert int(f[0].item()) == int(t[0].item())
    for a, b in zip(f[1:], t[1:]):
        a, b = a.cpu().numpy(), b.cpu().numpy()
        np.testing.assert_allclose(a, b, rtol=RTOL, atol=1e-9 * max(1.0, np.nanmax(np.abs(b))) if np.isfinite(b).any() else 0)


@pytest.mark.parametrize("kind", ["sorted_offset", "one_class_first", "single_class", "huge_mean"])
def test_gda_fit_fallback(ml, kind):
    """Inputs whose first rows misrepresent the class means: the rank-1 correction would cancel
    the shifted scatter, the device-side certification rejects it and pass 2 on the exact
    means runs; results equal the two-pass path either way."""
    n, d = 20_000, 64
    x = dev_units(ml, n, d, seed=10)
    y = ml.rng_ints(n, 2, seed=10, first_draw=n * d)
    if kind == "sorted_offset":        # first 64 rows near 0, the rest near 1e4
        x[64:] += 1.0e4
    elif kind == "one_class_first":    # first 64 rows all class 1, far from the class-0 mean
        y[:64] = 1
        x[:64] -= 5.0e3
    elif kind == "single_class":       # class 0 empty: mu0 is NaN, S from class 1 only
        y[:] = 1
    else:                              # mean 1e6, unit spread: the shift handles it
        x += 1.0e6
    f = ml.gda_fit(x, y)
    fb = ml.gda_fit_last_fallback(x)
    if kind in ("sorted_offset", "one_class_first"):
        assert fb
    if kind == "huge_mean":
        assert not fb
    t = _gda_two_pass(ml, x, y)
    assert int(f[0].item()) == int(t[0].item())
    for a, b in zip(f[1:], t[1:]):
        a, b = a.cpu().numpy(), b.cpu().numpy()
        assert np.array_equal(np.isnan(a), np.isnan(b))
        fin = np.isfinite(b)
        if fin.any():
            np.testing.assert_allclose(a[fin], b[fin], rtol=RTOL, atol=1e-9 * np.abs(b[fin]).max())


@pytest.mark.parametrize("kind", ["late_outlier", "zero_first_tiles", "late_nan", "late_inf", "tiny_column"])
def test_gda_fit_int8_range(ml, kind):
    """The int8 fit quantises each column per CTA from its first tile: a later value outside
    that range (or inf / NaN) must force the exact pass 2, a column that is tiny everywhere must
    keep its relative precision; results equal the two-pass path either way."""
    n, d = 300_001, 64
    x = dev_units(ml, n, d, seed=13)
    y = ml.rng_ints(n, 2, seed=13, first_draw=n * d)
    assert ml.gda_fit_path(x, y) == "int8"
    if kind == "late_outlier":          # row 250,000: 1e7 in one column (first tiles: O(1))
        x[250_000, 5] = 1.0e7
    elif kind == "zero_first_tiles":    # column 3 constant over every CTA's first tile, then not
        x[:96 * 148 * 2, 3] = 0.5
    elif kind == "late_nan":
        x[200_000, 7] = float("nan")
    elif kind == "late_inf":
        x[123_456, 9] = float("inf")
    else:                               # column 11 at 1e-100 scale everywhere
        x[:, 11] *= 1.0e-100
    f = ml.gda_fit(x, y)
    fb = ml.gda_fit_last_fallback(x)
    if kind in ("late_outlier", "zero_first_tiles", "late_nan", "late_inf"):
        assert fb
    else:
        assert not fb
    t = _gda_two_pass(ml, x, y)
    assert int(f[0].item()) == int(t[0].item())
    for a, b in zip(f[1:], t[1:]):
        a, b = a.cpu().numpy(), b.cpu().numpy()
        assert np.array_equal(np.isnan(a), np.isnan(b))
        fin = np.isfinite(b)
        if fin.any():
            np.testing.assert_allclose(a[fin], b[fin], rtol=RTOL, atol=1e-9 * np.abs(b[fin]).max())
    if kind == "tiny_column":   # its own scale: row and column 11 of S against the two-pass S
        Sa, Sb = f[3].cpu().numpy(), t[3].cpu().numpy()
        np.testing.assert_allclose(Sa[11], Sb[11], rtol=RTOL, atol=1e-9 * np.abs(Sb[11]).max())


@pytest.mark.parametrize("n", [1_048_576, 300_001, 97, 1])
def test_gda_fit_int8_matches_dmma(ml, n, monkeypatch):
    """The int8 tensor-core fit and the DMMA fit (DLX_GDA_I8=0) on the same inputs: equal n1,
    means and scatter within the fp64 tolerance; both scatters bitwise symmetric."""
    d = 64
    x = dev_units(ml, n, d, seed=14)
    y = ml.rng_ints(n, 2, seed=14, first_draw=n * d)
    assert ml.gda_fit_path(x, y) == "int8"
    a = [t.cpu().numpy() for t in ml.gda_fit(x, y)]
    monkeypatch.setenv("DLX_GDA_I8", "0")
    assert ml.gda_fit_path(x, y) == "dmma"
    b = [t.cpu().numpy() for t in ml.gda_fit(x, y)]
    assert int(a[0]) == int(b[0])
    assert np.array_equal(a[3], a[3].T, equal_nan=True) and np.array_equal(b[3], b[3].T, equal_nan=True)
    for u, v in zip(a[1:], b[1:]):
        assert np.array_equal(np.isnan(u), np.isnan(v))
        fin = np.isfinite(v)
        if fin.any():
            np.testing.assert_allclose(u[fin], v[fin], rtol=RTOL, atol=1e-9 * np.abs(v[fin]).max())


# ---- generic collect / reduce -------------------------------------------------------------------------

def test_generic_families(ml):
    n = 1_000_003
    x = ml.rng_units(n, seed=11)
    y = ml.rng_units(n, seed=12)
    xh, yh = x.cpu().numpy(), y.cpu().numpy()
    assert np.array_equal(ml.map_axpy(2.5, x, y).cpu().numpy(), O.axpy(2.5, xh, yh))   # SPEC.md:642 exact
    np.testing.assert_allclose(ml.reduce_sum(x).item(), O.sum_f64(xh), rtol=1e-12)
    ints = torch.arange(1, 10 ** 6 + 1, dtype=torch.int64, device="cuda")
    assert ml.reduce_sum(ints).item() == 500000500000
    assert ml.count_where_gt(x * 10, 7.0).item() == O.count_gt_f64(xh * 10, 7.0)
    m, v = ml.mean_variance(x)
    s, sq = O.sum_sumsq_f64(xh)
    np.testing.assert_allclose([m, v], [s / n, sq / n - (s / n) ** 2], rtol=1e-9)
    m, v = ml.mean_variance(torch.full((1000,), 0.3, dtype=torch.float64, device="cuda"))
    assert abs(v) < 1e-12


def test_generation_failed_is_loud(ml):
    from paper_1109_0778_b200 import GenerationFailed
    x = dev_units(ml, 10, 129 * 4, seed=1)   # odd-size row groups beyond the row kernel plan
    y = ml.rng_ints(10, 2, seed=1)
    with pytest.raises(GenerationFailed):
        ml.logreg_grad(x, y, torch.zeros(129 * 4, dtype=torch.float64, device="cuda"))


@pytest.mark.parametrize("n,d,k,method", [(0, 16, 8, 0), (4096, 16, 8, 0), (20_000, 64, 64, 0),
                                          (300_001, 64, 64, 2), (5000, 30, 5, 1), (3000, 66, 9, 1),
                                          (2000, 16, 80, 1), (1003, 16, 8, 2)])
def test_kmeans_iteration_fused_update(ml, n, d, k, method):
    """dlx_kmeans_iteration (update fused into the combine launch) equals dlx_kmeans_step +
    dlx_kmeans_update bit for bit on every path (small, screened, direct, empty input)."""
    x = dev_units(ml, max(n, k), d, seed=11)[:n] if n else torch.empty((0, d), dtype=torch.float64, device="cuda")
    mu0 = dev_units(ml, k, d, seed=12)
    a, c, s = ml.kmeans_step(x, mu0, method=method)
    mu_ref = ml.kmeans_update(c, s)
    mu = mu0.clone()
    a2, c2, s2 = ml.kmeans_iteration(x, mu, method=method)
    assert torch.equal(c, c2) and torch.equal(s.view(torch.int64), s2.view(torch.int64))
    assert torch.equal(mu.view(torch.int64), mu_ref.view(torch.int64))
    if n:
        assert torch.equal(a, a2)
