"""The drop-in executor (include/dlx_program.h: dlx_program_create / _execute, the replacement of
the reference's missing interpret / executeDEG) on the BASELINE configs at full shape, against
SURVEY Appendix B and the oracle, plus the ExecOptions / RunResult surface: caller inputs
(host and device), the program's result Value, cached lowerings, and the device-side k-means
update group."""
import math

import numpy as np
import pytest

import oracle as O
from paper_1109_0778_b200 import descriptors as D

pytestmark = pytest.mark.gpu


def lines(text):
    return [s for s in text.split("\n") if s != ""]


def close(a, b, rtol=1e-9):
    return abs(a - b) <= rtol * max(abs(a), abs(b))


def test_c3_gda_through_the_dropin(golden):
    """BASELINE C3 (GDA, N = 1M, d = 64) as the reference stages it — pass 1 = 1 + 2d keyed
    reduces, pass 2 = d^2 scatter reduces — through dlx_program_execute: App. B's n1, mu0[0],
    mu1[0], S[0][0], S[0][1], S[63][63] and every printed value against the oracle
    (rtol 1e-9; n1 exact)."""
    from paper_1109_0778_b200.program import Program
    n, d = 1 << 20, 64
    r = Program(D.gda_program(n, d)).run(seed=1)
    assert [e["family"] for e in r.report] == ["bucket_rows", "gda_scatter"]
    out = lines(r.output)
    assert len(out) == 1 + 2 * d + d * d
    g = golden["c3_gda"]
    n1 = int(out[0])
    mu0 = np.array([float(v) for v in out[1:1 + 2 * d:2]])
    mu1 = np.array([float(v) for v in out[2:2 + 2 * d:2]])
    S = np.array([float(v) for v in out[1 + 2 * d:]]).reshape(d, d)
    assert n1 == g["n1"]
    assert close(mu0[0], float(g["mu0_0"])) and close(mu1[0], float(g["mu1_0"]))
    assert close(S[0, 0], float(g["S00"])) and close(S[0, 1], float(g["S01"])) and close(S[63, 63], float(g["S6363"]))
    x = O.rng_units(1, 0, n * d).reshape(n, d)
    y = O.rng_ints(1, n * d, n, 2)
    n1r, s0, s1 = O.gda_pass1(x, y, workers=O.threads(), chunks=4 * O.threads())
    m0, m1 = s0 / float(n - n1r), s1 / float(n1r)
    Sr = O.gda_pass2(x, y, m0, m1, workers=O.threads(), chunks=4 * O.threads())
    np.testing.assert_allclose(mu0, m0, rtol=1e-9, atol=0)
    np.testing.assert_allclose(mu1, m1, rtol=1e-9, atol=0)
    np.testing.assert_allclose(S, Sr, rtol=1e-9, atol=1e-9 * np.abs(Sr).max())


@pytest.mark.parametrize("n,d", [(20000, 4), (4097, 7), (1000, 66), (3, 64)])
def test_gda_program_shapes_against_oracle(n, d):
    """Odd d (scalar row loads), d > 64 (two column groups) and tiny n through the drop-in."""
    from paper_1109_0778_b200.program import Program
    r = Program(D.gda_program(n, d)).run(seed=3)
    out = lines(r.output)
    x = O.rng_units(3, 0, n * d).reshape(n, d)
    y = O.rng_ints(3, n * d, n, 2)
    n1r, s0, s1 = O.gda_pass1(x, y)
    m0, m1 = s0 / float(n - n1r), s1 / float(n1r)
    Sr = O.gda_pass2(x, y, m0, m1)
    assert int(out[0]) == n1r
    got = np.array([float(v) for v in out[1:]])
    exp = np.concatenate([np.stack([m0, m1], 1).reshape(-1), Sr.reshape(-1)])
    np.testing.assert_allclose(got, exp, rtol=1e-9, atol=1e-12 * max(1.0, np.abs(exp).max()))


def test_c1_kmeans_ten_iterations_device_update(golden):
    """C1 (65,536 x 16, k = 8, 10 iterations) as ONE staged program of 10 fused loops: every
    iteration's centroid update runs on the device (no host round trip between iterations);
    the counts of all 10 iterations equal App. B exactly and mu[0][0] after iteration 1."""
    from paper_1109_0778_b200.program import Program
    g = golden["c1_kmeans"]
    n, d, k, it = 65536, 16, 8, 10
    prog = Program(D.kmeans_program(n, d, k, it))
    r = prog.run(seed=1)
    assert all(e["family"] == "kmeans" and e["update"] == "device" for e in r.report)
    out = lines(r.output)
    per = 1 + k
    for t in range(it):
        assert [int(v) for v in out[t * per + 1:(t + 1) * per]] == g["counts"][t], t
    # the oracle's free-running 10 iterations: assignment of row 0 and final centroids
    x, mu0 = O.kmeans_inputs(n, d, k)
    hist = O.kmeans_run(x, k, it, mu0)
    for t in range(it):
        assert int(out[t * per]) == int(hist[t][4][0])
    mu = np.array([float(v) for v in out[it * per:]])
    np.testing.assert_allclose(mu, hist[-1][2].reshape(-1), rtol=1e-9, atol=0)
    # executed again: every loop's lowering comes from the handle's cache, same text
    r2 = prog.run(seed=1)
    assert all(e["cached"] for e in r2.report) and r2.output == r.output


def test_c4_kmeans_program_matches_family_api():
    """C4 (16M x 64, k = 64) through the drop-in for 3 iterations equals the family API's
    iterations bit for bit (assignment of row 0, counts, final centroids); iteration 1's
    counts prefix and mu[0][0] equal App. B."""
    import torch
    from paper_1109_0778_b200 import multiloops as ml
    from paper_1109_0778_b200.program import Program
    n, d, k, it = 16_777_216, 64, 64, 3
    r = Program(D.kmeans_program(n, d, k, it)).run(seed=1)
    assert all(e["update"] == "device" for e in r.report)
    out = lines(r.output)
    x = ml.rng_units(n * d, seed=1, device=torch.device("cuda")).view(n, d)
    mu = x[:k].clone()
    per = 1 + k
    for t in range(it):
        a, c, s = ml.kmeans_step(x, mu)
        assert int(out[t * per]) == int(a[0].item())
        assert [int(v) for v in out[t * per + 1:(t + 1) * per]] == c.cpu().tolist()
        mu = ml.kmeans_update(c, s)
    got = np.array([float(v) for v in out[it * per:]])
    assert np.array_equal(got.view(np.int64), mu.cpu().numpy().reshape(-1).view(np.int64))
    del x


def test_c2_logreg_twenty_iterations_through_the_dropin():
    """BASELINE C2 (logistic regression BGD, N = 1M, d = 64, 20 iterations) as ONE staged program
    of 20 fused loops (collect h = sigmoid(theta . x_i) + 64 gradient reduces, theta updated on
    the device): theta after 20 iterations and h(0) of every iteration against the family API
    (LogRegProgram, itself pinned to the oracle) at rtol 1e-9, and the first iteration's h(0)
    against the oracle."""
    import torch
    from paper_1109_0778_b200 import multiloops as ml
    from paper_1109_0778_b200.programs import LogRegProgram
    from paper_1109_0778_b200.program import Program
    n, d, it = 1 << 20, 64, 20
    r = Program(D.logreg_program(n, d, it, 1.0 / n, link="sigmoid")).run(seed=1)
    assert all(e["family"] == "logistic" and e["update"] == "device" for e in r.report)
    out = [float(v) for v in lines(r.output)]
    assert len(out) == it + d
    dev = torch.device("cuda")
    x = ml.rng_units(n * d, seed=1, device=dev).view(n, d)
    y = ml.rng_ints(n, 2, seed=1, first_draw=n * d, device=dev)
    prog = LogRegProgram(x, y, torch.zeros(d, dtype=torch.float64, device=dev), 1.0 / n)
    for t in range(it):
        h0 = 1.0 / (1.0 + math.exp(0.0 - float((prog.theta * x[0]).sum().item())))
        assert close(out[t], h0, rtol=1e-12), t
        prog.run(1)
    np.testing.assert_allclose(out[it:], prog.theta.cpu().numpy(), rtol=1e-9, atol=1e-15)


@pytest.mark.parametrize("K", [64, 4096])
def test_c5_groupby_1e9_keys_through_the_dropin(golden, K):
    """BASELINE C5 (1e9 keys) as the reference stages it (one loop of K count reduces keyed on
    keys(i) == b) through the drop-in: bit-exact against App. B (first, last, min, max)."""
    from paper_1109_0778_b200.program import Program
    r = Program(D.groupby_program(1_000_000_000, K)).run(seed=1)
    assert [e["family"] for e in r.report] == ["groupby"]
    c = [int(v) for v in lines(r.output)]
    g = golden["c5_groupby"]["by_k"][str(K)]
    assert len(c) == K and sum(c) == 1_000_000_000
    assert (c[0], c[-1], min(c), max(c)) == (g["first"], g["last"], g["min"], g["max"])


def _collect_program(n):
    """x = randVector(n); y = collect(i -> 2.5 * x(i)); s = sum(y); print s; result y."""
    B = D._Builder()
    root = []
    x = B.stmt(root, "VectorRand", "Vector[Double]", [B.i(n)])
    i, y = B.sym(), B.sym()
    body = []
    xv = B.stmt(body, "VectorApply", "Double", [B.s(x, "Vector[Double]"), B.s(i, "Int")])
    tv = B.stmt(body, "Times", "Double", [B.d(2.5), B.s(xv, "Double")])
    el = {"kind": "collect", "live": True, "out": y, "out_ty": "Vector[Double]", "elem": B.block(body, B.s(tv, "Double")),
          "cond": -1, "combine": -1, "append": False}
    B.stmts[str(y)] = {"op": "ParallelLoop", "ty": "Vector[Double]", "args": [],
                       "loop": {"range": B.i(n), "index": i, "body": B.block([], {"u": 1, "t": "Unit"}, bound=[i]),
                                "elems": [el]}}
    root.append(y)
    j, s = B.sym(), B.sym()
    body = []
    yv = B.stmt(body, "VectorApply", "Double", [B.s(y, "Vector[Double]"), B.s(j, "Int")])
    el = B.reduce_elem(s, "Double", B.block(body, B.s(yv, "Double")), -1, B.d(0.0))
    B.stmts[str(s)] = {"op": "ParallelLoop", "ty": "Double", "args": [],
                       "loop": {"range": B.i(n), "index": j, "body": B.block([], {"u": 1, "t": "Unit"}, bound=[j]),
                                "elems": [el]}}
    root.append(s)
    B.stmt(root, "Print", "Unit", [B.s(s, "Double")])
    B.blocks["0"] = {"stmts": root, "result": B.s(y, "Vector[Double]"), "bound": []}
    return {"format": "dlx-program/1", "root": 0, "stmts": B.stmts, "blocks": B.blocks}, x


def test_run_result_value_and_inputs():
    """RunResult.result (runtime.hpp:100-103) carries the program's result Value (a vector here,
    downloaded to the host); dlx_program_input replaces the program's random source with caller
    data from host memory or device memory (the draw counter still advances)."""
    import torch
    from paper_1109_0778_b200.program import Program
    n = 100_003
    desc, xsym = _collect_program(n)
    prog = Program(desc)
    r = prog.run(seed=7)
    xr = O.rng_units(7, 0, n)
    assert isinstance(r.result, np.ndarray) and r.result.dtype == np.float64
    assert np.array_equal(r.result, 2.5 * xr)
    assert close(float(lines(r.output)[0]), float((2.5 * xr).sum()))
    data = np.linspace(-1.0, 1.0, n)
    rh = prog.run(seed=7, inputs={xsym: data})
    assert np.array_equal(rh.result, 2.5 * data)
    dt = torch.tensor(data, device="cuda")
    rd = prog.run(seed=7, inputs={xsym: dt})
    assert np.array_equal(rd.result, 2.5 * data)
    assert torch.equal(dt.cpu(), torch.tensor(data))   # used in place, not modified
    from paper_1109_0778_b200 import DlxError
    with pytest.raises(DlxError):
        prog.run(inputs={xsym: data[:10]})   # length must match the statement


def test_prints_of_pending_results_keep_program_order():
    """The k-means iterations are enqueued back to back (their prints are filled in when the
    results arrive); the output equals the serialised execution line for line."""
    from paper_1109_0778_b200.program import Program
    prog = Program(D.kmeans_program(4096, 16, 8, 4))
    a = prog.run(seed=2)
    b = prog.run(seed=2, serial=True)
    c = prog.run(seed=2, no_cache=True)
    assert a.output == b.output == c.output
    assert max(e["in_flight"] for e in a.report) >= 1     # no host sync between iterations
    assert all(e["in_flight"] == 0 for e in b.report)
    assert not math.isnan(float(lines(a.output)[-1]))


def test_reference_side_binding_run_staged():
    """The C++ reference-side binding (integration/stagekit_dlx_run.cpp: run_on_b200, what a
    stagekit `run` pipeline calls instead of interpret / executeDEG) end to end: programs staged
    with the REFERENCE DSL, fused and scheduled by the reference's own passes, executed through
    dlx_program_create / _execute and compared with the reference's emitted MiniC evaluated on
    the CPU (oracle/_ref/run_staged, built from /root/reference by oracle/ref.mk where the
    reference exists; it ships prebuilt to the GPU box)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "run_staged")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/run_staged not built (no /root/reference where the repo was built)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS") == 4 and "FAIL" not in r.stdout, r.stdout


def test_parallel_print_formatting_two_threads():
    """Programs whose joined loops print > 256 values format them on the host pool
    (program.cpp: HostPool); two handles on two host threads (the e2e bench's pattern) give the
    serial formatting's text exactly, every run."""
    import os
    import subprocess
    import sys
    import threading
    from paper_1109_0778_b200.descriptors import gda_program
    from paper_1109_0778_b200.program import Program
    desc = gda_program(20000, 24)   # 24^2 + 2 * 24 + 1 = 625 printed values after the joins
    ref = Program(desc).run(seed=3).output
    progs = [Program(desc), Program(desc)]
    outs = [[], []]

    def work(t):
        for _ in range(4):
            outs[t].append(progs[t].run(seed=3).output)

    ths = [threading.Thread(target=work, args=(t,)) for t in range(2)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert all(o == ref for o in outs[0] + outs[1])
    # the serial path (DLX_HOST_POOL=0) prints the same text, and a process using the pool exits
    code = ("import sys; sys.path.insert(0, %r); from paper_1109_0778_b200.descriptors import gda_program; "
            "from paper_1109_0778_b200.program import Program; print(Program(gda_program(20000, 24)).run(seed=3).output, end='')"
            % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    for env_pool in ("0", "1"):
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                           env=dict(os.environ, DLX_HOST_POOL=env_pool))
        assert r.returncode == 0, r.stderr[-2000:]
        assert r.stdout == ref
