"""The generic lowering (paper_1109_0778_b200/csrc/lower_jit.cpp): a root multiloop outside the
specialised families becomes ONE kernel generated from the loop body and compiled by NVRTC for
sm_100a.  CPU tests compile the generated kernels (NVRTC needs no device); GPU tests run
programs the bytecode kernel (vm.cu, DLX_PROGRAM_VM=1) cannot — more than 16 elems, nested
reduces, a load guarded by IfThenElse — and compare with sequential restatements (bit-exact
values; reduces at rtol 1e-9 since only the combine order differs)."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
COMPILED_FIXTURES = ["axpy_n100000", "count_gt_n100000", "find_count_n100000", "mean_variance_n100000"]


def load(name):
    with open(os.path.join(HERE, "golden", "staged", name + ".json")) as f:
        return json.load(f)


def _program(build):
    from paper_1109_0778_b200.descriptors import _Builder
    B = _Builder()
    root = []
    build(B, root)
    B.blocks["0"] = {"stmts": root, "result": {"u": 1, "t": "Unit"}, "bound": []}
    return {"format": "dlx-program/1", "root": 0, "stmts": B.stmts, "blocks": B.blocks}


def _loop(B, root, n, index, elems, ty):
    out = elems[0]["out"]
    B.stmts[str(out)] = {"op": "ParallelLoop", "ty": ty, "args": [],
                         "loop": {"range": B.i(n), "index": index,
                                  "body": B.block([], {"u": 1, "t": "Unit"}, bound=[index]), "elems": elems}}
    root.append(out)
    return out


def many_sums_program(n, d):
    """x = randVector(n*d); ONE loop of d reduces s_j = sum_i x(i*d+j)^2 (d > 16: beyond the
    bytecode kernel's elem cap); every s_j printed."""
    def build(B, root):
        x = B.stmt(root, "VectorRand", "Vector[Double]", [B.i(n * d)])
        i = B.sym()
        elems = []
        for j in range(d):
            body = []
            row = B.stmt(body, "Times", "Int", [B.i(d), B.s(i, "Int")])
            ix = B.stmt(body, "Plus", "Int", [B.s(row, "Int"), B.i(j)])
            v = B.stmt(body, "VectorApply", "Double", [B.s(x, "Vector[Double]"), B.s(ix, "Int")])
            sq = B.stmt(body, "Times", "Double", [B.s(v, "Double"), B.s(v, "Double")])
            elems.append(B.reduce_elem(B.sym(), "Double", B.block(body, B.s(sq, "Double")), -1, B.d(0.0)))
        _loop(B, root, n, i, elems, "Double")
        for e in elems:
            B.stmt(root, "Print", "Unit", [B.s(e["out"], "Double")])
    return _program(build)


def row_norms_program(n, d):
    """x = randVector(n*d); h = collect(i -> sum_j x(i*d+j) * x(i*d+j)) (a nested reduce over
    j inside the collect elem), fused with t = sum_i h(i); prints h(0), h(n-1), t."""
    def build(B, root):
        x = B.stmt(root, "VectorRand", "Vector[Double]", [B.i(n * d)])
        i, j = B.sym(), B.sym()
        # inner reduce over j (the reference's nested mk_reduce)
        ib = []
        row = B.stmt(ib, "Times", "Int", [B.i(d), B.s(i, "Int")])
        ix = B.stmt(ib, "Plus", "Int", [B.s(row, "Int"), B.s(j, "Int")])
        v = B.stmt(ib, "VectorApply", "Double", [B.s(x, "Vector[Double]"), B.s(ix, "Int")])
        sq = B.stmt(ib, "Times", "Double", [B.s(v, "Double"), B.s(v, "Double")])
        inner_out = B.sym()
        inner = B.reduce_elem(inner_out, "Double", B.block(ib, B.s(sq, "Double")), -1, B.d(0.0))
        B.stmts[str(inner_out)] = {"op": "ParallelLoop", "ty": "Double", "args": [],
                                   "loop": {"range": B.i(d), "index": j,
                                            "body": B.block([], {"u": 1, "t": "Unit"}, bound=[j]),
                                            "elems": [inner]}}
        h = B.sym()
        col = {"kind": "collect", "live": True, "out": h, "out_ty": "Vector[Double]",
               "elem": B.block([inner_out], B.s(inner_out, "Double")), "cond": -1, "combine": -1, "append": False}
        tot = B.reduce_elem(B.sym(), "Double", B.block([inner_out], B.s(inner_out, "Double")), -1, B.d(0.0))
        _loop(B, root, n, i, [col, tot], "Vector[Double]")
        for k in (0, n - 1):
            a = B.stmt(root, "VectorApply", "Double", [B.s(h, "Vector[Double]"), B.i(k)])
            B.stmt(root, "Print", "Unit", [B.s(a, "Double")])
        B.stmt(root, "Print", "Unit", [B.s(tot["out"], "Double")])
    return _program(build)


def guarded_load_program(n, m):
    """v = randVector(m); s = sum_{i < n} (if (i < m) v(i) else 0.0) with n > m: the load runs
    only on the taken branch (MiniC `if`), so no index traps."""
    def build(B, root):
        v = B.stmt(root, "VectorRand", "Vector[Double]", [B.i(m)])
        i = B.sym()
        body = []
        lt = B.stmt(body, "Lt", "Bool", [B.s(i, "Int"), B.i(m)])
        tb = []
        ld = B.stmt(tb, "VectorApply", "Double", [B.s(v, "Vector[Double]"), B.s(i, "Int")])
        sel = B.stmt(body, "IfThenElse", "Double", [B.s(lt, "Bool")],
                     blocks=[B.block(tb, B.s(ld, "Double")), B.block([], B.d(0.0))])
        el = B.reduce_elem(B.sym(), "Double", B.block(body, B.s(sel, "Double")), -1, B.d(0.0))
        _loop(B, root, n, i, [el], "Double")
        B.stmt(root, "Print", "Unit", [B.s(el["out"], "Double")])
    return _program(build)


def int_mix_program(n):
    """keys = randIntVector(n, 1000); one loop of Int reduces with wraparound products, a
    predicated count and a bool collect: p = prod_i (2 * key(i) + 1) (wraps), c = #{key < 10},
    b(i) = key(i) == 7; prints p, c, b(0)."""
    def build(B, root):
        k = B.stmt(root, "VectorRandInt", "Vector[Int]", [B.i(n), B.i(1000)])
        i = B.sym()
        b1 = []
        kv = B.stmt(b1, "VectorApply", "Int", [B.s(k, "Vector[Int]"), B.s(i, "Int")])
        t = B.stmt(b1, "Times", "Int", [B.i(2), B.s(kv, "Int")])
        o = B.stmt(b1, "Plus", "Int", [B.s(t, "Int"), B.i(1)])
        prod = B.reduce_elem(B.sym(), "Int", B.block(b1, B.s(o, "Int")), -1, B.i(1))
        l, r = B.sym(), B.sym()   # product combine: Times(rv_left, rv_right)
        cb = []
        pm = B.stmt(cb, "Times", "Int", [B.s(l, "Int"), B.s(r, "Int")])
        prod.update(combine=B.block(cb, B.s(pm, "Int"), bound=[l, r]), rv_left=l, rv_right=r)
        cc = []
        kv2 = B.stmt(cc, "VectorApply", "Int", [B.s(k, "Vector[Int]"), B.s(i, "Int")])
        lt = B.stmt(cc, "Lt", "Bool", [B.s(kv2, "Int"), B.i(10)])
        cnt = B.reduce_elem(B.sym(), "Int", B.block([], B.i(1)), B.block(cc, B.s(lt, "Bool")), B.i(0))
        bb = []
        kv3 = B.stmt(bb, "VectorApply", "Int", [B.s(k, "Vector[Int]"), B.s(i, "Int")])
        eq = B.stmt(bb, "Eq", "Bool", [B.s(kv3, "Int"), B.i(7)])
        bc = {"kind": "collect", "live": True, "out": B.sym(), "out_ty": "Vector[Bool]",
              "elem": B.block(bb, B.s(eq, "Bool")), "cond": -1, "combine": -1, "append": False}
        _loop(B, root, n, i, [prod, cnt, bc], "Int")
        B.stmt(root, "Print", "Unit", [B.s(prod["out"], "Int")])
        B.stmt(root, "Print", "Unit", [B.s(cnt["out"], "Int")])
        a = B.stmt(root, "VectorApply", "Bool", [B.s(bc["out"], "Vector[Bool]"), B.i(0)])
        B.stmt(root, "Print", "Unit", [B.s(a, "Bool")])
    return _program(build)


def lines(text):
    return [s for s in text.split("\n") if s != ""]


# ---- CPU: lowering + NVRTC compile (no device) -------------------------------------------------

@pytest.mark.parametrize("name", COMPILED_FIXTURES)
def test_staged_generic_loops_compile(name, monkeypatch):
    """The reference-staged programs outside the specialised families: every loop is lowered to
    a generated kernel that NVRTC compiles for sm_100a."""
    from paper_1109_0778_b200.program import run_program
    monkeypatch.setenv("DLX_PROGRAM_DRYRUN", "1")
    monkeypatch.setenv("DLX_PROGRAM_DRYRUN_COMPILE", "1")
    _, report = run_program(load(name)["program"], seed=1)
    assert report and all(r["family"] == "compiled" for r in report)


@pytest.mark.parametrize("prog", ["many_sums", "row_norms", "guarded_load", "int_mix"])
def test_beyond_vm_caps_compile(prog, monkeypatch):
    from paper_1109_0778_b200.program import run_program
    p = {"many_sums": lambda: many_sums_program(1000, 40), "row_norms": lambda: row_norms_program(1000, 12),
         "guarded_load": lambda: guarded_load_program(100, 10), "int_mix": lambda: int_mix_program(1000)}[prog]()
    monkeypatch.setenv("DLX_PROGRAM_DRYRUN", "1")
    monkeypatch.setenv("DLX_PROGRAM_DRYRUN_COMPILE", "1")
    _, report = run_program(p, seed=1)
    assert [r["family"] for r in report] == ["compiled"]
    # the bytecode kernel cannot take them (elem cap, nested reduce) — except the guarded load
    monkeypatch.setenv("DLX_PROGRAM_VM", "1")
    if prog in ("many_sums", "row_norms"):
        from paper_1109_0778_b200 import GenerationFailed
        import subprocess
        import sys
        # DLX_PROGRAM_VM is read once per process: check in a fresh one
        code = ("import json,sys; sys.path.insert(0, %r); sys.path.insert(0, %r);"
                "from paper_1109_0778_b200.program import run_program;"
                "from test_compiled_loops import many_sums_program, row_norms_program;"
                "p = %s; run_program(p, seed=1)") % (os.path.dirname(HERE), HERE,
                                                     "many_sums_program(1000, 40)" if prog == "many_sums"
                                                     else "row_norms_program(1000, 12)")
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                           env=dict(os.environ, DLX_PROGRAM_VM="1", DLX_PROGRAM_DRYRUN="1"))
        assert r.returncode != 0 and "GenerationFailed" in r.stderr
        del GenerationFailed


# ---- GPU ---------------------------------------------------------------------------------------

def _same(a, b, rtol=1e-9):
    fa, fb = float(a), float(b)
    return fa == fb or abs(fa - fb) <= rtol * max(abs(fa), abs(fb))


@pytest.mark.gpu
def test_many_sums_on_b200():
    from paper_1109_0778_b200.program import run_program
    n, d = 200_003, 40
    text, report = run_program(many_sums_program(n, d), seed=1)
    assert [r["family"] for r in report] == ["compiled"]
    x = O.rng_units(1, 0, n * d).reshape(n, d)
    exp = (x * x).sum(axis=0)
    got = [float(v) for v in lines(text)]
    assert all(_same(g, e) for g, e in zip(got, exp)) and len(got) == d


@pytest.mark.gpu
def test_row_norms_nested_reduce_on_b200():
    """The collect's nested reduce folds left in j with rounded products (no FMA): h(i) is
    bit-identical to the sequential restatement; the total matches at rtol."""
    from paper_1109_0778_b200.program import run_program
    n, d = 100_001, 12
    text, report = run_program(row_norms_program(n, d), seed=1)
    assert [r["family"] for r in report] == ["compiled"]
    x = O.rng_units(1, 0, n * d).reshape(n, d)
    h = np.zeros(n)
    for j in range(d):   # sequential in j, one rounding per op (numpy: no contraction)
        h = h + x[:, j] * x[:, j]
    got = lines(text)
    assert got[0] == O.format_double(h[0]) and got[1] == O.format_double(h[-1])
    assert _same(got[2], h.sum())


@pytest.mark.gpu
def test_guarded_load_on_b200():
    from paper_1109_0778_b200.program import run_program
    text, _ = run_program(guarded_load_program(1000, 10), seed=1)
    v = O.rng_units(1, 0, 10)
    assert _same(lines(text)[0], v.sum())


@pytest.mark.gpu
def test_int_mix_on_b200():
    from paper_1109_0778_b200.program import run_program
    n = 300_007
    text, _ = run_program(int_mix_program(n), seed=1)
    k = O.rng_ints(1, 0, n, 1000).astype(np.uint64)
    p = np.uint64(1)
    with np.errstate(over="ignore"):
        for v in (2 * k + 1):   # wraparound product (mod 2^64), order-free
            p = p * v
    got = lines(text)
    assert int(got[0]) == int(np.int64(p.astype(np.int64)))
    assert int(got[1]) == int((k < 10).sum())
    assert got[2] == ("true" if k[0] == 7 else "false")


@pytest.mark.gpu
@pytest.mark.parametrize("name", COMPILED_FIXTURES)
def test_compiled_equals_bytecode_kernel(name):
    """The generated kernel and the bytecode kernel (DLX_PROGRAM_VM=1, a fresh process) print
    the same text for the reference-staged programs both can run."""
    import subprocess
    import sys
    from paper_1109_0778_b200.program import run_program
    fx = load(name)
    text, _ = run_program(fx["program"], seed=1)
    code = ("import json,sys; sys.path.insert(0, %r);"
            "from paper_1109_0778_b200.program import run_program;"
            "fx = json.load(open(%r)); print(run_program(fx['program'], seed=1)[0], end='')") % (
        os.path.dirname(HERE), os.path.join(HERE, "golden", "staged", name + ".json"))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                       env=dict(os.environ, DLX_PROGRAM_VM="1"))
    assert r.returncode == 0, r.stderr
    assert lines(r.stdout) == lines(text) or all(_same(a, b) for a, b in zip(lines(r.stdout), lines(text)))
