"""Directly built descriptors (paper_1109_0778_b200/descriptors.py) against the programs the
REFERENCE's own staging + fuse_loops + schedule produce (tests/golden/staged/*.json, made by
oracle/_ref/stage_programs from /root/reference/proj): statement by statement, after renaming
every symbol by first appearance, the two descriptors must be the same program.  This pins the
production-shape builders (used where the reference's quadratic fusion pass cannot stage C3 /
C4-sized programs) to what the reference itself would hand the executor."""
import json
import os

import pytest

from paper_1109_0778_b200 import descriptors as D

HERE = os.path.dirname(os.path.abspath(__file__))


def load(name):
    with open(os.path.join(HERE, "golden", "staged", name + ".json")) as f:
        return json.load(f)["program"]


def canon(p):
    """The program as text with symbols renamed in traversal order (blocks inline)."""
    names = {}

    def nm(s):
        if s not in names:
            names[s] = f"v{len(names)}"
        return names[s]

    out = []

    def atom(a):
        if "s" in a:
            return nm(a["s"]) + ":" + a.get("t", "")
        if "d" in a:
            return f"{a['d']!r}d"
        if "i" in a:
            return f"{a['i']}i"
        if "b" in a:
            return f"{a['b']}b"
        return "u"

    def block(b, ind):
        bl = p["blocks"][str(b)]
        for s in bl["stmts"]:
            stmt(s, ind)
        out.append(ind + "-> " + atom(bl["result"]))

    def stmt(s, ind):
        st = p["stmts"][str(s)]
        out.append(ind + f"{nm(s)} = {st['op']}:{st['ty']}({','.join(atom(a) for a in st['args'])})"
                   + (f" aux={st['aux_ty']}" if "aux_ty" in st else ""))
        for b in st.get("blocks", []):
            block(b, ind + "  ")
        if "loop" in st:
            lp = st["loop"]
            out.append(ind + f"  range {atom(lp['range'])} index {nm(lp['index'])}")
            block(lp["body"], ind + "  ")
            for e in lp["elems"]:
                out.append(ind + f"  elem {e['kind']} live={e['live']} append={e['append']} out={nm(e['out'])}:"
                           f"{e['out_ty']} zero={atom(e['zero']) if 'zero' in e else '-'}")
                for k in ("cond", "elem", "combine"):
                    if e[k] >= 0:
                        if k == "combine":
                            out.append(ind + f"   rv {nm(e['rv_left'])} {nm(e['rv_right'])}")
                        out.append(ind + "   " + k)
                        block(e[k], ind + "    ")

    block(p["root"], "")
    return out


def first_diff(a, b):
    for q, (x, y) in enumerate(zip(a, b)):
        if x != y:
            return q, x, y
    return min(len(a), len(b)), None, None


def test_gda_program_is_the_reference_staged_program():
    got, exp = canon(D.gda_program(20000, 4)), canon(load("gda_n20000_d4"))
    assert got == exp, first_diff(got, exp)


def test_groupby_program_is_the_reference_staged_program():
    got, exp = canon(D.groupby_program(100000, 16)), canon(load("groupby_n100000_k16"))
    assert got == exp, first_diff(got, exp)


def test_logreg_program_is_the_reference_staged_program():
    got = canon(D.logreg_program(20000, 8, 2, 1.0 / 20000, link="softsign"))
    exp = canon(load("logreg_n20000_d8_it2"))
    assert got == exp, first_diff(got, exp)


@pytest.mark.parametrize("link", ["softsign", "sigmoid"])
def test_logreg_program_c2_lowers_to_logistic_with_device_update(link):
    """C2 (N = 1M, d = 64, 20 BGD iterations) through the drop-in: every iteration's fused loop
    (1 collect + 64 gradient reduces) lowers to the logistic family and its 64 host updates
    theta(j) = theta(j) - alpha * g_j run on the device (UpdateGroup::Axpy)."""
    from paper_1109_0778_b200.program import Program
    n, d, it = 1 << 20, 64, 20
    r = Program(D.logreg_program(n, d, it, 1.0 / n, link=link)).run(dry_run=True)
    assert [e["family"] for e in r.report] == ["logistic"] * it
    assert all(e["update"] == "device" and e["live_elems"] == 1 + d for e in r.report)


@pytest.mark.parametrize("name,shape", [("kmeans_n4096_d16_k8_it2", (4096, 16, 8, 2)),
                                        ("kmeans_n65536_d16_k8_it1", (65536, 16, 8, 1))])
def test_kmeans_program_is_the_reference_staged_program(name, shape):
    got, exp = canon(D.kmeans_program(*shape)), canon(load(name))
    assert got == exp, first_diff(got, exp)


def test_gda_program_c3_lowers_to_bucket_rows_and_scatter():
    """C3 (N = 1M, d = 64) through the drop-in: pass 1 (1 + 2d = 129 keyed reduces) lowers to
    the bucket-row-sum kernel, pass 2 (d^2 = 4,096 reduces) to the DMMA scatter — no
    GenerationFailed at d >= 8 (the round-1 interpreter's 16-elem cap)."""
    from paper_1109_0778_b200.program import Program
    r = Program(D.gda_program(1 << 20, 64)).run(dry_run=True)
    assert [e["family"] for e in r.report] == ["bucket_rows", "gda_scatter"]
    assert r.report[0]["live_elems"] == 129 and r.report[0]["buckets"] == 2 and r.report[0]["d"] == 64
    assert r.report[1]["live_elems"] == 4096 and r.report[1]["d"] == 64


@pytest.mark.parametrize("shape", [(4096, 16, 8, 2), (65536, 16, 8, 10), (16_777_216, 64, 64, 3)])
def test_kmeans_program_update_group_on_device(shape):
    """Every iteration's k*d host statements mu(c*d+j) = sum_cj / toDouble(count_c)
    (vectordsl.cpp:90-103) are recognised as one update group and run on the device in the
    loop's combine launch (dlx_kmeans_iteration)."""
    from paper_1109_0778_b200.program import Program
    n, d, k, it = shape
    r = Program(D.kmeans_program(n, d, k, it)).run(dry_run=True)
    assert [e["family"] for e in r.report] == ["kmeans"] * it
    assert all(e["update"] == "device" and e["launch"] == "dlx_kmeans_iteration" for e in r.report)


def test_update_group_not_fused_when_mu_is_read_in_between():
    """A read of mu between the loop and its updates must see the old centroids, so the group
    stays on the host (the analysis refuses it)."""
    from paper_1109_0778_b200.program import Program
    p = D.kmeans_program(4096, 16, 8, 1)
    root = p["blocks"]["0"]["stmts"]
    loop = next(q for q, s in enumerate(root) if p["stmts"][str(s)]["op"] == "ParallelLoop")
    mu = next(int(k) for k, s in p["stmts"].items() if s["op"] == "VectorNew")
    new = max(int(k) for k in p["stmts"]) + 1
    p["stmts"][str(new)] = {"op": "VectorApply", "ty": "Double", "args": [{"s": mu, "t": "Vector[Double]"}, {"i": 3, "t": "Int"}]}
    p["stmts"][str(new + 1)] = {"op": "Print", "ty": "Unit", "args": [{"s": new, "t": "Double"}]}
    root[loop + 1:loop + 1] = [new, new + 1]
    r = Program(p).run(dry_run=True)
    assert r.report[0]["family"] == "kmeans" and r.report[0]["launch"] == "dlx_kmeans_step"


def test_nonfinite_literals_round_trip():
    """Double literals the reference constant-folds to inf / nan (graph.cpp:211-216) travel as
    "inf" / "-inf" / "nan" strings (JSON numbers cannot hold them) and print as the reference's
    format_double does."""
    import math
    from paper_1109_0778_b200.program import Program
    B = D._Builder()
    root = []
    for v in (math.inf, -math.inf, math.nan, 1.5):
        B.stmt(root, "Print", "Unit", [B.d(v)])
    B.blocks["0"] = {"stmts": root, "result": {"u": 1, "t": "Unit"}, "bound": []}
    prog = {"format": "dlx-program/1", "root": 0, "stmts": B.stmts, "blocks": B.blocks}
    assert '"inf"' in json.dumps(prog) and '"nan"' in json.dumps(prog)
    r = Program(prog).run(dry_run=True)
    assert r.output.split() == ["inf", "-inf", "nan", "1.5"]


@pytest.mark.parametrize("link", ["sigmoid", "softsign"])
def test_logistic_link_runs_as_fixed_function(link, monkeypatch):
    """The link compiled from the staged loop body (1 / (1 + exp(0 - t)), t / (1 + |t|)) is
    recognised and evaluated by the fixed functor, not the per-row interpreter (csrc/rows.cu
    link_kind); the reference-staged logreg fixture carries the softsign."""
    import json
    from paper_1109_0778_b200 import descriptors as D
    from paper_1109_0778_b200.program import run_program
    monkeypatch.setenv("DLX_PROGRAM_DRYRUN", "1")
    _, rep = run_program(D.logreg_program(1000, 8, 2, 0.001, link=link), seed=1)
    assert [r["link"] for r in rep] == [link, link]
    if link == "softsign":
        fx = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "staged", "logreg_n20000_d8_it2.json")))
        assert [r["link"] for r in run_program(fx["program"], seed=1)[1]] == ["softsign", "softsign"]
