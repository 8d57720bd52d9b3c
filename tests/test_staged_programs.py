"""Programs staged through the REFERENCE's own DSL, fusion and codegen (oracle/_ref build of
/root/reference/proj, integration/stage_programs.cpp), with expected output produced by
executing the reference's emitted MiniC (oracle/minic_eval.hpp).  CPU tests pin those
fixtures against the oracle port; GPU tests run the same descriptors through the B200
executor (dlx_program_run) and compare with the reference's output."""
import glob
import json
import math
import os

import numpy as np
import pytest

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
FIXTURES = sorted(glob.glob(os.path.join(HERE, "golden", "staged", "*.json")))


def load(name):
    with open(os.path.join(HERE, "golden", "staged", name + ".json")) as f:
        return json.load(f)


def lines(text):
    return [s for s in text.split("\n") if s != ""]


def same_value(a: str, b: str, rtol=1e-9) -> bool:
    if a == b:
        return True
    try:
        ia, ib = int(a), int(b)
        return ia == ib
    except ValueError:
        pass
    fa, fb = float(a), float(b)
    if math.isnan(fa) and math.isnan(fb):
        return True
    return abs(fa - fb) <= rtol * max(abs(fa), abs(fb))


def test_fixtures_present():
    names = {os.path.basename(f)[:-5] for f in FIXTURES}
    for n in ("kmeans_n65536_d16_k8_it1", "kmeans_n4096_d16_k8_it2", "kmeans_n4096_d16_k8_it2_assign",
              "groupby_n100000_k16", "gda_n20000_d4",
              "logreg_n20000_d8_it2",
              "mean_variance_n100000", "axpy_n100000", "count_gt_n100000", "find_count_n100000"):
        assert n in names
    for f in FIXTURES:
        with open(f) as fh:
            fx = json.load(fh)
        assert fx["program"]["format"] == "dlx-program/1"
        assert fx["expected"]


def test_staged_kmeans_matches_appendix_b(golden):
    fx = load("kmeans_n65536_d16_k8_it1")
    out = lines(fx["expected"])
    assert [int(v) for v in out[1:9]] == golden["c1_kmeans"]["counts"][0]
    assert out[9] == golden["c1_kmeans"]["mu00"][0]
    assert fx["root_loops"] == 1  # one fused multiloop per iteration


def test_staged_kmeans_matches_oracle_port():
    fx = load("kmeans_n4096_d16_k8_it2")
    x, mu0 = O.kmeans_inputs(4096, 16, 8)
    hist = O.kmeans_run(x, 8, 2, mu0)
    exp = lines(fx["expected"])
    got = []
    for counts, _, _, _, assign in hist:
        got.append(str(int(assign[0])))
        got += [str(int(c)) for c in counts]
    got += [O.format_double(v) for v in hist[-1][2].reshape(-1)]
    assert exp == got


def test_staged_kmeans_every_assignment_matches_oracle_port():
    """The reference-staged program that prints the WHOLE assignment vector after each of its two
    iterations (integration/stage_programs.cpp kmeans(..., all_assign)): the oracle's assignments
    equal, element by element, what the reference's own emitted MiniC computes."""
    fx = load("kmeans_n4096_d16_k8_it2_assign")
    n, d, k = 4096, 16, 8
    x, mu0 = O.kmeans_inputs(n, d, k)
    hist = O.kmeans_run(x, k, 2, mu0)
    exp = lines(fx["expected"])
    got = []
    for counts, _, _, _, assign in hist:
        got += [str(int(a)) for a in assign]
        got += [str(int(c)) for c in counts]
    got += [O.format_double(v) for v in hist[-1][2].reshape(-1)]
    assert len(exp) == 2 * (n + k) + k * d
    assert exp == got


def test_staged_groupby_gda_stats_match_oracle_port():
    exp = lines(load("groupby_n100000_k16")["expected"])
    keys = O.rng_ints(1, 0, 100000, 16)
    assert [int(v) for v in exp] == O.groupby_count(keys, 16).tolist()
    exp = lines(load("gda_n20000_d4")["expected"])
    n, d = 20000, 4
    x = O.rng_units(1, 0, n * d).reshape(n, d)
    y = O.rng_ints(1, n * d, n, 2)
    n1, s0, s1 = O.gda_pass1(x, y)
    mu0, mu1 = s0 / float(n - n1), s1 / float(n1)
    S = O.gda_pass2(x, y, mu0, mu1)
    got = [str(n1)] + [O.format_double(v) for pair in zip(mu0, mu1) for v in pair] + [O.format_double(v) for v in S.reshape(-1)]
    assert exp == got
    exp = lines(load("mean_variance_n100000")["expected"])
    xv = O.rng_units(1, 0, 100000)
    s, sq = O.sum_sumsq_f64(xv)
    mean = s / 100000
    assert exp[0] == O.format_double(mean)
    assert same_value(exp[1], O.format_double(sq / 100000 - mean * mean), rtol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(f)[:-5] for f in FIXTURES])
def test_staged_program_on_b200(path):
    from paper_1109_0778_b200.program import run_program
    with open(path) as f:
        fx = json.load(f)
    text, report = run_program(fx["program"], seed=fx["seed"])
    got, exp = lines(text), lines(fx["expected"])
    assert len(got) == len(exp)
    bad = [(i, g, e) for i, (g, e) in enumerate(zip(got, exp)) if not same_value(g, e)]
    assert not bad, bad[:5]
    fams = [r["family"] for r in report]
    print(os.path.basename(path), fams)
    name = os.path.basename(path)
    if name.startswith("kmeans"):
        assert "kmeans" in fams
    if name.startswith("groupby"):
        assert fams == ["groupby"]
    if name.startswith("gda"):
        assert fams == ["bucket_rows", "gda_scatter"]
    if name.startswith("logreg"):
        assert fams and set(fams) == {"logistic"} and all(r["update"] == "device" for r in report)


@pytest.mark.gpu
def test_unlowerable_loop_fails_loudly():
    from paper_1109_0778_b200 import GenerationFailed
    from paper_1109_0778_b200.program import run_program
    fx = load("count_gt_n100000")
    prog = json.loads(json.dumps(fx["program"]))
    # turn the loop's first live elem into a foreach (effectful disjoint writes): not lowered
    for st in prog["stmts"].values():
        if "loop" in st:
            st["loop"]["elems"][0]["kind"] = "foreach"
            break
    with pytest.raises(GenerationFailed):
        run_program(prog, seed=1)


def _patch_literal(prog, old, new):
    """Replace a double literal of the staged descriptor (the filter threshold)."""
    txt = json.dumps(prog)
    assert txt.count(json.dumps(old)) >= 1
    return json.loads(txt.replace(json.dumps(old), json.dumps(new)))


def _find_count_expected(n, thr):
    import numpy as np
    import oracle as O
    x = O.rng_units(1, 0, n)
    hits = np.nonzero(thr < x)[0]
    return hits


@pytest.mark.gpu
@pytest.mark.parametrize("thr", [0.9, 0.5, -1.0, 0.9999])
def test_filter_collect_thresholds(thr):
    """Filter-collect (append) through the generic kernel's ordered compaction: every
    selected index, in index order, for sparse / half / all-selected filters."""
    from paper_1109_0778_b200.program import run_program
    prog = _patch_literal(load("find_count_n100000")["program"], 0.9, thr)
    text, report = run_program(prog, seed=1)
    hits = _find_count_expected(100000, thr)
    got = lines(text)
    assert [int(v) for v in got] == [len(hits), len(hits), int(hits[0]), int(hits.sum())]
    assert [r["family"] for r in report] == ["compiled", "compiled"]


@pytest.mark.gpu
def test_filter_collect_empty_traps_on_read():
    """Nothing selected: the appended vector is empty and reading element 0 traps
    (TrapIndexOutOfBounds, as the reference's x(0) on an empty builder)."""
    from paper_1109_0778_b200 import TrapError
    from paper_1109_0778_b200.program import run_program
    prog = _patch_literal(load("find_count_n100000")["program"], 0.9, 2.0)
    with pytest.raises(TrapError):
        run_program(prog, seed=1)


EXPECTED_FAMILIES = {
    "axpy_n100000": ["compiled", "compiled"],
    "count_gt_n100000": ["compiled"],
    "find_count_n100000": ["compiled", "compiled"],
    "gda_n20000_d4": ["bucket_rows", "gda_scatter"],
    "groupby_n100000_k16": ["groupby"],
    "kmeans_n4096_d16_k8_it2": ["kmeans", "kmeans"],
    "kmeans_n65536_d16_k8_it1": ["kmeans"],
    "logreg_n20000_d8_it2": ["logistic", "logistic"],
    "mean_variance_n100000": ["compiled"],
}


@pytest.mark.parametrize("name", sorted(EXPECTED_FAMILIES))
def test_lowering_families_dry_run(name, monkeypatch):
    """CPU: parse + symbolically evaluate + match every loop of the reference-staged program
    (DLX_PROGRAM_DRYRUN: no device memory, no launches) and check the lowering chosen."""
    from paper_1109_0778_b200.program import run_program
    monkeypatch.setenv("DLX_PROGRAM_DRYRUN", "1")
    _, report = run_program(load(name)["program"], seed=1)
    assert [r["family"] for r in report] == EXPECTED_FAMILIES[name]


def _offset_program(p, off):
    """Renumber every symbol and block of a dlx-program/1 descriptor by `off`."""
    def atom(a):
        return dict(a, s=a["s"] + off) if "s" in a else a

    stmts = {}
    for k, st in p["stmts"].items():
        st = dict(st, args=[atom(a) for a in st["args"]])
        if "blocks" in st:
            st["blocks"] = [b + off for b in st["blocks"]]
        if "loop" in st:
            lp = st["loop"]
            lp = dict(lp, range=atom(lp["range"]), index=lp["index"] + off, body=lp["body"] + off)
            lp["elems"] = [dict(e, out=e["out"] + off, elem=e["elem"] + off,
                                cond=e["cond"] + off if e["cond"] >= 0 else -1,
                                combine=e["combine"] + off if e["combine"] >= 0 else -1,
                                rv_left=e.get("rv_left", -1) + off if e.get("rv_left", -1) >= 0 else -1,
                                rv_right=e.get("rv_right", -1) + off if e.get("rv_right", -1) >= 0 else -1)
                           for e in lp["elems"]]
            st["loop"] = lp
        stmts[str(int(k) + off)] = st
    blocks = {str(int(k) + off): dict(b, stmts=[s + off for s in b["stmts"]], result=atom(b["result"]),
                                      bound=[s + off for s in b.get("bound", [])])
              for k, b in p["blocks"].items()}
    return {"format": p["format"], "root": p["root"] + off, "stmts": stmts, "blocks": blocks}


def _merge_independent(pa, pb, off=100000):
    """One program running `pa` and a renumbered copy of `pb` side by side: each program's
    statements before its first loop, then both first loops back to back (no data edge between
    them in the DEG), then the rest of `pa`, then the rest of `pb`."""
    pb = _offset_program(pb, off)
    stmts = dict(pa["stmts"], **pb["stmts"])
    blocks = dict(pa["blocks"], **pb["blocks"])
    ra = pa["blocks"][str(pa["root"])]["stmts"]
    rb = pb["blocks"][str(pb["root"])]["stmts"]

    def split(root, st):
        i = next(q for q, s in enumerate(root) if st[str(s)]["op"] == "ParallelLoop")
        return root[:i], root[i], root[i + 1:]

    a0, la, a1 = split(ra, stmts)
    b0, lb, b1 = split(rb, stmts)
    root = a0 + b0 + [la, lb] + a1 + b1
    blocks[str(pa["root"])] = dict(blocks[str(pa["root"])], stmts=root)
    del blocks[str(pb["root"])]
    return {"format": pa["format"], "root": pa["root"], "stmts": stmts, "blocks": blocks}


def test_merged_program_lowers_both_loops_dry_run(monkeypatch):
    from paper_1109_0778_b200.program import run_program
    monkeypatch.setenv("DLX_PROGRAM_DRYRUN", "1")
    mv = load("mean_variance_n100000")["program"]
    _, report = run_program(_merge_independent(mv, mv), seed=1)
    assert [r["family"] for r in report] == ["compiled", "compiled"]


@pytest.mark.gpu
@pytest.mark.parametrize("second", ["mean_variance_n100000", "groupby_n100000_k16", "kmeans_n65536_d16_k8_it1"])
def test_independent_loops_overlap(second, monkeypatch):
    """DEG overlap (scheduleDEG): two root loops with no data edge between
    them run on different loop streams with the first still in flight when the second
    launches; results equal the serialised execution (DLX_PROGRAM_SERIAL) bit for bit and the
    first program's output equals its reference-staged fixture."""
    from paper_1109_0778_b200.program import run_program
    fa = load("mean_variance_n100000")
    merged = _merge_independent(fa["program"], load(second)["program"])
    text, report = run_program(merged, seed=1)
    assert len(report) == 2
    assert report[0]["in_flight"] == 0 and report[1]["in_flight"] == 1
    assert report[0]["stream"] != report[1]["stream"]
    monkeypatch.setenv("DLX_PROGRAM_SERIAL", "1")
    text_s, report_s = run_program(merged, seed=1)
    assert all(r["in_flight"] == 0 for r in report_s)
    assert text == text_s
    exp = lines(fa["expected"])
    assert all(same_value(g, e) for g, e in zip(lines(text)[:len(exp)], exp))
    if second == "mean_variance_n100000":   # the copy draws the next 100000 units
        x = O.rng_units(1, 100000, 100000)
        mean = x.sum() / 1e5
        got = lines(text)[len(exp):]
        assert same_value(got[0], repr(float(mean)))
        assert same_value(got[1], repr(float((x * x).sum() / 1e5 - mean * mean)))


@pytest.mark.parametrize("shape", [(4096, 16, 8, 2), (16_777_216, 64, 64, 1)])
def test_direct_kmeans_descriptor_dry_run(shape, monkeypatch):
    """CPU: the directly built k-means program (descriptors.kmeans_program: the reference's
    fused-loop shape without its quadratic fusion pass) lowers every iteration to the k-means
    family with all k(d+1)+1 elems live — at the fixture shape and at C4."""
    from paper_1109_0778_b200.descriptors import kmeans_program
    from paper_1109_0778_b200.program import run_program
    monkeypatch.setenv("DLX_PROGRAM_DRYRUN", "1")
    n, d, k, it = shape
    _, report = run_program(kmeans_program(n, d, k, it), seed=1)
    assert [r["family"] for r in report] == ["kmeans"] * it
    assert all(r["live_elems"] == 1 + k * (d + 1) and r["k"] == k and r["d"] == d for r in report)


@pytest.mark.gpu
@pytest.mark.parametrize("name,shape", [("kmeans_n4096_d16_k8_it2", (4096, 16, 8, 2)),
                                        ("kmeans_n65536_d16_k8_it1", (65536, 16, 8, 1))])
def test_direct_kmeans_descriptor_matches_reference_staged(name, shape):
    """The directly built program prints what the REFERENCE-staged program's MiniC prints
    (assignment of row 0, counts, every centroid) on the B200 executor."""
    from paper_1109_0778_b200.descriptors import kmeans_program
    from paper_1109_0778_b200.program import run_program
    text, report = run_program(kmeans_program(*shape), seed=1)
    got, exp = lines(text), lines(load(name)["expected"])
    assert len(got) == len(exp)
    assert all(same_value(g, e) for g, e in zip(got, exp))
    assert [r["family"] for r in report] == ["kmeans"] * shape[3]


def _two_trapping_loops():
    """Two independent root loops that both trap on the device: the first divides by zero
    (Int, at i = 5), the second loads past the end of a 10-element vector."""
    from paper_1109_0778_b200.descriptors import _Builder
    B = _Builder()
    root = []
    v = B.stmt(root, "VectorNew", "Vector[Double]", [B.i(10)], aux_ty="Double")
    outs = []
    for kind in ("div", "oob"):
        i, out = B.sym(), B.sym()
        body = []
        if kind == "div":
            m = B.stmt(body, "Minus", "Int", [B.s(i, "Int"), B.i(5)])
            q = B.stmt(body, "Divide", "Int", [B.i(1), B.s(m, "Int")])
            el = B.reduce_elem(out, "Int", B.block(body, B.s(q, "Int")), -1, B.i(0))
        else:
            ix = B.stmt(body, "Plus", "Int", [B.s(i, "Int"), B.i(1000)])
            q = B.stmt(body, "VectorApply", "Double", [B.s(v, "Vector[Double]"), B.s(ix, "Int")])
            el = B.reduce_elem(out, "Double", B.block(body, B.s(q, "Double")), -1, B.d(0.0))
        B.stmts[str(out)] = {"op": "ParallelLoop", "ty": el["out_ty"], "args": [],
                             "loop": {"range": B.i(100), "index": i, "body": B.block([], {"u": 1, "t": "Unit"}, bound=[i]),
                                      "elems": [el]}}
        root.append(out)
        outs.append(out)
    for o, ty in zip(outs, ("Int", "Double")):
        B.stmt(root, "Print", "Unit", [B.s(o, ty)])
    B.blocks["0"] = {"stmts": root, "result": {"u": 1, "t": "Unit"}, "bound": []}
    return {"format": "dlx-program/1", "root": 0, "stmts": B.stmts, "blocks": B.blocks}


def test_two_trapping_loops_dry_run(monkeypatch):
    from paper_1109_0778_b200.program import run_program
    monkeypatch.setenv("DLX_PROGRAM_DRYRUN", "1")
    _, report = run_program(_two_trapping_loops(), seed=1)
    assert [r["family"] for r in report] == ["compiled", "compiled"]


def _one_loop_two_traps(off):
    """One root loop over i < 100 with two reduce elems: the first divides by (i - 5) (Int),
    the second loads v(i + off) from a 10-element vector (out of range from i = 10 - off)."""
    from paper_1109_0778_b200.descriptors import _Builder
    B = _Builder()
    root = []
    v = B.stmt(root, "VectorNew", "Vector[Double]", [B.i(10)], aux_ty="Double")
    i, out = B.sym(), B.sym()
    b1, b2 = [], []
    m = B.stmt(b1, "Minus", "Int", [B.s(i, "Int"), B.i(5)])
    q = B.stmt(b1, "Divide", "Int", [B.i(1), B.s(m, "Int")])
    e1 = B.reduce_elem(out, "Int", B.block(b1, B.s(q, "Int")), -1, B.i(0))
    ix = B.stmt(b2, "Plus", "Int", [B.s(i, "Int"), B.i(off)])
    ld = B.stmt(b2, "VectorApply", "Double", [B.s(v, "Vector[Double]"), B.s(ix, "Int")])
    e2 = B.reduce_elem(B.sym(), "Double", B.block(b2, B.s(ld, "Double")), -1, B.d(0.0))
    B.stmts[str(out)] = {"op": "ParallelLoop", "ty": "Int", "args": [],
                         "loop": {"range": B.i(100), "index": i, "body": B.block([], {"u": 1, "t": "Unit"}, bound=[i]),
                                  "elems": [e1, e2]}}
    root.append(out)
    B.stmt(root, "Print", "Unit", [B.s(out, "Int")])
    B.stmt(root, "Print", "Unit", [B.s(e2["out"], "Double")])
    B.blocks["0"] = {"stmts": root, "result": {"u": 1, "t": "Unit"}, "bound": []}
    return {"format": "dlx-program/1", "root": 0, "stmts": B.stmts, "blocks": B.blocks}


@pytest.mark.gpu
@pytest.mark.parametrize("off,expect", [(7, "TrapIndexOutOfBounds.*index 3"),    # i=3 loads v(10) first
                                        (5, "TrapDivByZero.*index 5"),          # same index: elem 1 runs first
                                        (4, "TrapDivByZero.*index 5")])         # i=5 divides before i=6 loads
def test_first_trap_in_index_order(off, expect):
    """The reported trap is the one sequential interpret meets first: lowest index, then program
    order inside the index (codegen.cpp:391-425), whatever order the device threads trap in."""
    from paper_1109_0778_b200 import TrapError
    from paper_1109_0778_b200.program import run_program
    with pytest.raises(TrapError, match=expect):
        run_program(_one_loop_two_traps(off), seed=1)


@pytest.mark.gpu
@pytest.mark.parametrize("serial", [False, True])
def test_trap_of_earlier_loop_wins(serial, monkeypatch):
    """With both loops in flight, the earlier loop's trap (program order) is the one raised,
    as in sequential execution (Int division by zero traps)."""
    from paper_1109_0778_b200 import TrapError
    from paper_1109_0778_b200.program import run_program
    if serial:
        monkeypatch.setenv("DLX_PROGRAM_SERIAL", "1")
    with pytest.raises(TrapError, match="division by zero"):
        run_program(_two_trapping_loops(), seed=1)
    # the executor's per-device resources (loop streams, events, pinned staging) stay usable
    fx = load("mean_variance_n100000")
    text, _ = run_program(fx["program"], seed=1)
    assert all(same_value(g, e) for g, e in zip(lines(text), lines(fx["expected"])))


# ---- the executor's own fusion pass (csrc/fuse.cpp) --------------------
# Fixtures *_unfused are the same reference-staged programs with the reference's fuse_loops
# skipped (integration/stage_programs.cpp): the executor fuses their root (and nested) loops.
UNFUSED = sorted(os.path.basename(f)[:-len("_unfused.json")] for f in FIXTURES if f.endswith("_unfused.json"))
C4_UNFUSED = os.path.join(HERE, "golden", "staged_c4", "kmeans_n16777216_d64_k64_it1_unfused.program.json.xz")


def _strip(report):
    return [{k: v for k, v in e.items() if k not in ("loop", "cached")} for e in report]


def test_unfused_fixtures_present():
    assert set(UNFUSED) >= {"kmeans_n4096_d16_k8_it2", "groupby_n100000_k16", "gda_n20000_d4",
                            "logreg_n20000_d8_it2", "mean_variance_n100000", "find_count_n100000",
                            "axpy_n100000", "count_gt_n100000", "fusion_blockers_n10000"}


@pytest.mark.parametrize("name", UNFUSED)
def test_executor_fusion_matches_reference_fusion_dry_run(name, monkeypatch):
    """CPU: the unfused reference-staged program, fused by the executor, lowers loop for loop
    like the program the reference's fuse_loops fused (families, live elems, shapes, update
    placement); the unfused program's own MiniC output equals the fused one's."""
    from paper_1109_0778_b200.program import run_program
    monkeypatch.setenv("DLX_PROGRAM_DRYRUN", "1")
    fused, unf = load(name), load(name + "_unfused")
    assert unf["program"]["fusion"] == "executor" and unf["fused_pairs"] == 0
    assert unf["root_loops"] >= fused["root_loops"]
    assert fused["expected"] == unf["expected"]
    _, ra = run_program(fused["program"], seed=1)
    _, rb = run_program(unf["program"], seed=1)
    if name == "fusion_blockers_n10000":
        # the pairs the fusion must refuse stay apart: the two sums of m around its update, x's
        # sum and the map that reads it, loops of different ranges; the map and its own sum
        # (range VectorLength of the map) fuse vertically, which the reference never does
        assert [(e["n"], e["live_elems"]) for e in ra] == [(8, 1), (8, 1), (10000, 1), (10000, 1), (10000, 1), (5000, 1)]
        assert [(e["n"], e["live_elems"]) for e in rb] == [(8, 1), (8, 1), (10000, 1), (10000, 2), (5000, 1)]
        return
    if name == "axpy_n100000":
        # vertical fusion through VectorLength: z = zip_with(x, y) and z.sum() (range
        # VectorLength(z)) become ONE loop here; the reference's cycle check never lets its
        # vertical rule fire (the VectorLength statement is an intermediate, fusion.cpp:229)
        assert [e["family"] for e in ra] == ["compiled", "compiled"]
        assert [(e["family"], e["live_elems"]) for e in rb] == [("compiled", 2)]
        return
    assert _strip(ra) == _strip(rb)


def test_executor_fusion_c4_shape_dry_run(monkeypatch):
    """CPU: the headline program (one k-means iteration at N=16M, d=k=64) staged through the
    reference DSL WITHOUT the reference's fuse_loops (4,161 root loops; the reference's own
    fusion of it did not finish in 25 min) fuses in the executor into the one k-means
    multiloop with all 4,161 elems live, the centroid update on the device."""
    import lzma
    import time
    from paper_1109_0778_b200.program import Program
    monkeypatch.setenv("DLX_PROGRAM_DRYRUN", "1")
    with lzma.open(C4_UNFUSED, "rt") as f:
        text = f.read()
    p = json.loads(text)
    root = p["blocks"][str(p["root"])]["stmts"]
    assert p["fusion"] == "executor"
    assert sum(p["stmts"][str(s)]["op"] == "ParallelLoop" for s in root) == 4161
    t0 = time.time()
    r = Program(text).run(dry_run=True)
    assert time.time() - t0 < 60
    assert len(r.report) == 1
    e = r.report[0]
    assert (e["family"], e["live_elems"], e["n"], e["d"], e["k"], e["update"]) == \
        ("kmeans", 4161, 16_777_216, 64, 64, "device")


@pytest.mark.gpu
def test_executor_fusion_c4_shape_on_b200():
    """B200: the unfused C4 program fused by the executor prints exactly what the directly built
    C4 descriptor (descriptors.kmeans_program, pinned to the reference-staged fixtures) prints:
    the assignment of row 0, the 64 counts and all 4,096 updated centroids."""
    import lzma
    from paper_1109_0778_b200.descriptors import kmeans_program
    from paper_1109_0778_b200.program import Program
    with lzma.open(C4_UNFUSED, "rt") as f:
        got = Program(f.read()).run(seed=1)
    exp = Program(kmeans_program(16_777_216, 64, 64, 1)).run(seed=1)
    assert [r["family"] for r in got.report] == ["kmeans"]
    g, e = lines(got.output), lines(exp.output)
    assert len(g) == len(e) == 1 + 64 + 64 * 64
    assert g == e


# ---- the headline shape (d = k = 64) staged by the reference, unfused, at N = 4,096 -------------
HEADLINE_UNFUSED = os.path.join(HERE, "golden", "staged_c4", "kmeans_n4096_d64_k64_it2_unfused.json.xz")


def _load_xz(path):
    import lzma
    with lzma.open(path, "rt") as f:
        return json.load(f)


def test_headline_shape_unfused_fixture_matches_oracle_port():
    """Two k-means iterations at d = k = 64 staged through the reference DSL (8,322 root loops; the
    reference's fuse_loops cannot fuse this shape in reasonable time) and evaluated as the
    reference's own MiniC: the oracle port prints exactly the same text."""
    fx = _load_xz(HEADLINE_UNFUSED)
    assert fx["program"]["fusion"] == "executor" and fx["root_loops"] == 8322
    x, mu0 = O.kmeans_inputs(4096, 64, 64)
    hist = O.kmeans_run(x, 64, 2, mu0)
    got = []
    for counts, _, _, _, assign in hist:
        got.append(str(int(assign[0])))
        got += [str(int(c)) for c in counts]
    got += [O.format_double(v) for v in hist[-1][2].reshape(-1)]
    assert lines(fx["expected"]) == got


def test_headline_shape_unfused_dry_run(monkeypatch):
    """CPU: the executor fuses the 8,322 root loops into the two k-means multiloops (4,161 live
    elems each, centroid update on the device)."""
    from paper_1109_0778_b200.program import Program
    monkeypatch.setenv("DLX_PROGRAM_DRYRUN", "1")
    r = Program(_load_xz(HEADLINE_UNFUSED)["program"]).run(dry_run=True)
    assert [(e["family"], e["live_elems"], e["d"], e["k"], e["update"]) for e in r.report] == \
        [("kmeans", 4161, 64, 64, "device")] * 2


@pytest.mark.gpu
def test_headline_shape_unfused_on_b200():
    """B200: the unfused headline-shape program, fused by the executor and run on the tcgen05
    screened kernel, prints the reference MiniC's output (ints exact, doubles rtol 1e-9)."""
    from paper_1109_0778_b200.program import Program
    fx = _load_xz(HEADLINE_UNFUSED)
    r = Program(fx["program"]).run(seed=fx["seed"])
    got, exp = lines(r.output), lines(fx["expected"])
    assert len(got) == len(exp) == 2 * 65 + 64 * 64
    bad = [(i, g, e) for i, (g, e) in enumerate(zip(got, exp)) if not same_value(g, e)]
    assert not bad, bad[:5]
