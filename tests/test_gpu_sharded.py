"""Multi-device execution of the drop-in (ExecOptions.devices; paper_1109_0778_b200/csrc/shard.cpp):
every root loop of a sharded family runs as contiguous index shards, one per listed device, and
the shards' partial records are folded in ascending shard order (executeDEG's ascending-chunk
combine).  The pool's boxes have one GPU, so the shards share device 0; with
DLX_SHARD_REPLICATE=1 every shard also takes the cross-device path (its input windows drawn by
LCG skip-ahead or peer-copied, its outputs peer-copied back), exactly as on a multi-GPU node.

Parity: integer outputs (assignments, counts, GroupBy) bit-exact and fp64 values rtol 1e-9
against the single-device run of the same program, the reference-staged fixtures' expected text,
and the oracle."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def load(name):
    with open(os.path.join(HERE, "golden", "staged", name + ".json")) as f:
        return json.load(f)


def lines(text):
    return [s for s in text.split("\n") if s != ""]


def same(a, b, rtol=1e-9):
    if a == b:
        return True
    try:
        return int(a) == int(b)
    except ValueError:
        pass
    fa, fb = float(a), float(b)
    if math.isnan(fa) and math.isnan(fb):
        return True
    return abs(fa - fb) <= rtol * max(abs(fa), abs(fb))


SHARDED_FIXTURES = ["kmeans_n4096_d16_k8_it2", "kmeans_n65536_d16_k8_it1", "kmeans_n4096_d16_k8_it2_assign",
                    "groupby_n100000_k16", "gda_n20000_d4", "logreg_n20000_d8_it2"]


@pytest.mark.parametrize("replicate", [False, True])
@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("name", SHARDED_FIXTURES)
def test_sharded_fixture(name, G, replicate, monkeypatch):
    from paper_1109_0778_b200.program import Program
    if replicate:
        monkeypatch.setenv("DLX_SHARD_REPLICATE", "1")
    fx = load(name)
    prog = Program(fx["program"])
    r = prog.run(seed=1, devices=[0] * G)
    assert all(e.get("shards") == G for e in r.report), r.report
    exp = lines(fx["expected"])
    got = lines(r.output)
    assert len(got) == len(exp)
    assert all(same(g, e) for g, e in zip(got, exp))
    one = lines(prog.run(seed=1).output)
    ints = [(g, o) for g, o in zip(got, one) if "." not in o and "e" not in o and "n" not in o]
    assert all(g == o for g, o in ints)   # integer lines (assignments, counts) bit-exact


@pytest.mark.parametrize("replicate", [False, True])
def test_sharded_kmeans_c4_shape(replicate, monkeypatch):
    """d = k = 64 (the screened tcgen05 kernel per shard), 4 shards of 300,001 uneven rows, three
    fused iterations with the centroid update fused into the ascending-shard fold."""
    from paper_1109_0778_b200 import descriptors as D
    from paper_1109_0778_b200.program import Program
    if replicate:
        monkeypatch.setenv("DLX_SHARD_REPLICATE", "1")
    n, d, k, it = 300_001, 64, 64, 3
    prog = Program(D.kmeans_program(n, d, k, it))
    r4 = prog.run(seed=1, devices=[0, 0, 0, 0])
    assert [e["family"] for e in r4.report] == ["kmeans"] * it
    assert all(e["shards"] == 4 and e["update"] == "device" for e in r4.report)
    x, mu = O.kmeans_inputs(n, d, k)
    hist = O.kmeans_run(x, k, it, mu, workers=O.threads(), chunks=4 * O.threads())
    got = lines(r4.output)
    per = 1 + k
    for t, (counts, _, _, _, assign) in enumerate(hist):
        assert int(got[t * per]) == int(assign[0])
        assert [int(v) for v in got[t * per + 1:(t + 1) * per]] == counts.tolist()
    np.testing.assert_allclose(np.array([float(v) for v in got[it * per:]]), hist[-1][2].reshape(-1), rtol=1e-9)


@pytest.mark.parametrize("G", [2, 5])
def test_sharded_gda_logreg_groupby_programs(G, monkeypatch):
    """C3 / C2 / C5 shapes (smaller N) through the sharded drop-in with the cross-device path."""
    from paper_1109_0778_b200 import descriptors as D
    from paper_1109_0778_b200.program import Program
    monkeypatch.setenv("DLX_SHARD_REPLICATE", "1")
    devs = [0] * G
    for desc, fams in ((D.gda_program(100_003, 64), ["bucket_rows", "gda_scatter"]),
                       (D.logreg_program(60_001, 64, 3, 1.0 / 60_001), ["logistic"] * 3),
                       (D.groupby_program(1_000_003, 4096), ["groupby"])):
        prog = Program(desc)
        rs = prog.run(seed=1, devices=devs)
        r1 = prog.run(seed=1)
        assert [e["family"] for e in rs.report] == fams
        assert all(e["shards"] == G for e in rs.report)
        a, b = lines(rs.output), lines(r1.output)
        assert len(a) == len(b) and all(same(u, v) for u, v in zip(a, b))


def test_bad_device_is_an_argument_error():
    from paper_1109_0778_b200.program import Program
    from paper_1109_0778_b200._lib import DlxError
    prog = Program(load("groupby_n100000_k16")["program"])
    with pytest.raises(DlxError, match="not a device"):
        prog.run(seed=1, devices=[0, 4096])
