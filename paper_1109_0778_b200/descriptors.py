"""Direct construction of "dlx-program/1" descriptors for the OptiML k-means iteration, in the
shape the reference's own staging produces ("production callers may construct a
LoopPayload-shaped descriptor directly — no staging/fusion at 4k-elem scale").

The reference front-end stages one k-means iteration as ONE fused ParallelLoop (fuse_loops,
proj/src/fusion.cpp:170-288): a collect whose elem is the staged_if argmin chain over k inner
distance reduces (stage.cpp:73-104; loops.cpp:111-174), horizontally fused with the k counts
and k*d sums, each a predicated reduce keyed on the collect's value (vertical fusion
substitutes it), then host statements mu(c*d+j) = sum_cj / toDouble(count_c)
(vectordsl.cpp:90-103).  At the headline shape (k = d = 64: 4,160 elems) the reference's
fusion pass is quadratic, so this module emits the same loop payload
(node.hpp:60-81: range, index, body, elems with elem / cond / combine blocks, zero,
rv_left / rv_right) without it.  `tests/test_staged_programs.py` checks that the directly built
program at the fixture shape produces exactly the reference-staged program's output.
"""
from __future__ import annotations

import json
import math


class _Builder:
    def __init__(self):
        self.stmts: dict[str, dict] = {}
        self.blocks: dict[str, dict] = {}
        self.next_sym = 0
        self.next_block = 1   # block 0 is the root

    @staticmethod
    def s(sym: int, ty: str) -> dict:
        return {"s": sym, "t": ty}

    @staticmethod
    def i(v: int) -> dict:
        return {"i": int(v), "t": "Int"}

    @staticmethod
    def d(v: float) -> dict:
        v = float(v)
        if v != v:   # non-finite literals as strings (JSON numbers cannot hold them)
            return {"d": "-nan" if math.copysign(1.0, v) < 0 else "nan", "t": "Double"}
        if v in (math.inf, -math.inf):
            return {"d": "inf" if v > 0 else "-inf", "t": "Double"}
        return {"d": v, "t": "Double"}

    def sym(self) -> int:
        self.next_sym += 1
        return self.next_sym - 1

    def stmt(self, out: list, op: str, ty: str, args: list, **extra) -> int:
        x = self.sym()
        self.stmts[str(x)] = dict(op=op, ty=ty, args=args, **extra)
        out.append(x)
        return x

    def block(self, stmts: list, result: dict, bound=()) -> int:
        b = self.next_block
        self.next_block += 1
        self.blocks[str(b)] = {"stmts": stmts, "result": result, "bound": list(bound)}
        return b

    def reduce_elem(self, out: int, ty: str, elem: int, cond: int, zero: dict) -> dict:
        l, r = self.sym(), self.sym()
        body = []
        p = self.stmt(body, "Plus", ty, [self.s(l, ty), self.s(r, ty)])
        comb = self.block(body, self.s(p, ty), bound=[l, r])
        return {"kind": "reduce", "live": True, "out": out, "out_ty": ty, "elem": elem, "cond": cond,
                "combine": comb, "append": False, "zero": zero, "rv_left": l, "rv_right": r}


def kmeans_program(n: int, d: int, k: int, iters: int = 1) -> dict:
    """The staged program of integration/stage_programs.cpp::kmeans(n, d, k, iters): x =
    randVector(n*d), mu = the first k rows of x, `iters` fused iterations (each prints the
    assignment of row 0 and the k counts), then the k*d centroids are printed."""
    B = _Builder()
    root: list[int] = []
    VD, VI = "Vector[Double]", "Vector[Int]"
    x = B.stmt(root, "VectorRand", VD, [B.i(n * d)])
    mu = B.stmt(root, "VectorNew", VD, [B.i(k * d)], aux_ty="Double")
    for e in range(k * d):
        a = B.stmt(root, "VectorApply", "Double", [B.s(x, VD), B.i(e)])
        B.stmt(root, "VectorUpdate", "Unit", [B.s(mu, VD), B.i(e), B.s(a, "Double")])
    for _ in range(iters):
        i = B.sym()                       # the loop index
        loop_sym = B.sym()                # the collect's out (= the ParallelLoop statement)
        # collect elem: k distance reduces over j (one fused inner loop), then the argmin chain
        eb: list[int] = []
        j = B.sym()
        douts = [B.sym() for _ in range(k)]
        inner_elems = []
        row = None
        for c in range(k):
            body: list[int] = []
            if row is None:   # i*d is CSE'd: defined in the first distance elem, reused by the rest
                row = B.stmt(body, "Times", "Int", [B.i(d), B.s(i, "Int")])
            xi = B.stmt(body, "Plus", "Int", [B.s(row, "Int"), B.s(j, "Int")])
            xv = B.stmt(body, "VectorApply", "Double", [B.s(x, VD), B.s(xi, "Int")])
            mi = j if c == 0 else B.stmt(body, "Plus", "Int", [B.i(c * d), B.s(j, "Int")])
            mv = B.stmt(body, "VectorApply", "Double", [B.s(mu, VD), B.s(mi, "Int")])
            df = B.stmt(body, "Minus", "Double", [B.s(xv, "Double"), B.s(mv, "Double")])
            sq = B.stmt(body, "Times", "Double", [B.s(df, "Double"), B.s(df, "Double")])
            inner_elems.append(B.reduce_elem(douts[c], "Double", B.block(body, B.s(sq, "Double")), -1, B.d(0.0)))
        inner_body = B.block([], {"u": 1, "t": "Unit"}, bound=[j])
        B.stmts[str(douts[0])] = {"op": "ParallelLoop", "ty": "Double", "args": [],
                                  "loop": {"range": B.i(d), "index": j, "body": inner_body, "elems": inner_elems}}
        eb.append(douts[0])
        best, idx = B.d(1e300), B.i(0)
        for c in range(k):
            lt = B.stmt(eb, "Lt", "Bool", [B.s(douts[c], "Double"), best])
            if c + 1 < k:   # the last best is dead (the reference's DCE drops it)
                nb = B.stmt(eb, "IfThenElse", "Double", [B.s(lt, "Bool")],
                            blocks=[B.block([], B.s(douts[c], "Double")), B.block([], best)])
            ni = B.stmt(eb, "IfThenElse", "Int", [B.s(lt, "Bool")],
                        blocks=[B.block([], B.i(c)), B.block([], idx)])
            if c + 1 < k:
                best = B.s(nb, "Double")
            idx = B.s(ni, "Int")
        a_sym = idx["s"]
        elems = [{"kind": "collect", "live": True, "out": loop_sym, "out_ty": VI, "elem": B.block(eb, idx),
                  "cond": -1, "combine": -1, "append": False}]
        counts, sums = [], []
        for c in range(k):
            def cond_block():
                cb: list[int] = []
                q = B.stmt(cb, "Eq", "Bool", [B.s(a_sym, "Int"), B.i(c)])
                return B.block(cb, B.s(q, "Bool"))
            cnt = B.sym()
            counts.append(cnt)
            elems.append(B.reduce_elem(cnt, "Int", B.block([], B.i(1)), cond_block(), B.i(0)))
            for jj in range(d):
                body = []
                row = B.stmt(body, "Times", "Int", [B.i(d), B.s(i, "Int")])
                xi = row if jj == 0 else B.stmt(body, "Plus", "Int", [B.i(jj), B.s(row, "Int")])
                xv = B.stmt(body, "VectorApply", "Double", [B.s(x, VD), B.s(xi, "Int")])
                sm = B.sym()
                sums.append(sm)
                elems.append(B.reduce_elem(sm, "Double", B.block(body, B.s(xv, "Double")), cond_block(), B.d(0.0)))
        body = B.block([], {"u": 1, "t": "Unit"}, bound=[i])
        B.stmts[str(loop_sym)] = {"op": "ParallelLoop", "ty": VI, "args": [],
                                  "loop": {"range": B.i(n), "index": i, "body": body, "elems": elems}}
        root.append(loop_sym)
        a0 = B.stmt(root, "VectorApply", "Int", [B.s(loop_sym, VI), B.i(0)])
        B.stmt(root, "Print", "Unit", [B.s(a0, "Int")])
        for c in range(k):
            B.stmt(root, "Print", "Unit", [B.s(counts[c], "Int")])
            cd = B.stmt(root, "ToDouble", "Double", [B.s(counts[c], "Int")])
            for jj in range(d):
                q = B.stmt(root, "Divide", "Double", [B.s(sums[c * d + jj], "Double"), B.s(cd, "Double")])
                B.stmt(root, "VectorUpdate", "Unit", [B.s(mu, VD), B.i(c * d + jj), B.s(q, "Double")])
    for e in range(k * d):
        v = B.stmt(root, "VectorApply", "Double", [B.s(mu, VD), B.i(e)])
        B.stmt(root, "Print", "Unit", [B.s(v, "Double")])
    B.blocks["0"] = {"stmts": root, "result": {"u": 1, "t": "Unit"}, "bound": []}
    return {"format": "dlx-program/1", "root": 0, "stmts": B.stmts, "blocks": B.blocks}


def gda_program(n: int, d: int) -> dict:
    """The staged program of integration/stage_programs.cpp::gda(n, d) in the shape the reference's
    staging + fusion produce (tests/test_descriptors.py compares it statement by statement with
    the reference-staged gda_n20000_d4 fixture): x = randVector(n*d), y = randIntVector(n, 2);
    pass 1 = ONE fused loop of a count (y(i) == 1) and 2d column sums keyed on y(i) == 0 / 1
    (loops.cpp:111-174); the means on the host; pass 2 = ONE fused loop of d*d reduces
    (x(i*d+a) - mean_{y_i,a}) * (x(i*d+b) - mean_{y_i,b}) with IfThenElse mean selects; every
    value printed."""
    B = _Builder()
    root: list[int] = []
    VD, VI = "Vector[Double]", "Vector[Int]"
    x = B.stmt(root, "VectorRand", VD, [B.i(n * d)])
    y = B.stmt(root, "VectorRandInt", VI, [B.i(n), B.i(2)])

    def key_cond(i, c):
        cb: list[int] = []
        yi = B.stmt(cb, "VectorApply", "Int", [B.s(y, VI), B.s(i, "Int")])
        q = B.stmt(cb, "Eq", "Bool", [B.s(yi, "Int"), B.i(c)])
        return B.block(cb, B.s(q, "Bool"))

    # pass 1
    i = B.sym()
    n1 = B.sym()
    elems = [B.reduce_elem(n1, "Int", B.block([], B.i(1)), key_cond(i, 1), B.i(0))]
    s0, s1 = [], []
    for j in range(d):
        for c, outl in ((0, s0), (1, s1)):
            body: list[int] = []
            row = B.stmt(body, "Times", "Int", [B.i(d), B.s(i, "Int")])
            ix = row if j == 0 else B.stmt(body, "Plus", "Int", [B.i(j), B.s(row, "Int")])
            xv = B.stmt(body, "VectorApply", "Double", [B.s(x, VD), B.s(ix, "Int")])
            o = B.sym()
            outl.append(o)
            elems.append(B.reduce_elem(o, "Double", B.block(body, B.s(xv, "Double")), key_cond(i, c), B.d(0.0)))
    B.stmts[str(n1)] = {"op": "ParallelLoop", "ty": "Int", "args": [],
                        "loop": {"range": B.i(n), "index": i, "body": B.block([], {"u": 1, "t": "Unit"}, bound=[i]),
                                 "elems": elems}}
    root.append(n1)
    nn1 = B.stmt(root, "ToDouble", "Double", [B.s(n1, "Int")])
    m0 = B.stmt(root, "Minus", "Int", [B.i(n), B.s(n1, "Int")])
    nn0 = B.stmt(root, "ToDouble", "Double", [B.s(m0, "Int")])
    mu0, mu1 = [], []
    for j in range(d):
        mu0.append(B.stmt(root, "Divide", "Double", [B.s(s0[j], "Double"), B.s(nn0, "Double")]))
        mu1.append(B.stmt(root, "Divide", "Double", [B.s(s1[j], "Double"), B.s(nn1, "Double")]))
    B.stmt(root, "Print", "Unit", [B.s(n1, "Int")])
    for j in range(d):
        B.stmt(root, "Print", "Unit", [B.s(mu0[j], "Double")])
        B.stmt(root, "Print", "Unit", [B.s(mu1[j], "Double")])
    # pass 2
    i2 = B.sym()
    outs, elems = [], []
    for a in range(d):
        for b in range(d):
            body = []
            yi = B.stmt(body, "VectorApply", "Int", [B.s(y, VI), B.s(i2, "Int")])
            c1 = B.stmt(body, "Eq", "Bool", [B.s(yi, "Int"), B.i(1)])
            ma = B.stmt(body, "IfThenElse", "Double", [B.s(c1, "Bool")],
                        blocks=[B.block([], B.s(mu1[a], "Double")), B.block([], B.s(mu0[a], "Double"))])
            mb = B.stmt(body, "IfThenElse", "Double", [B.s(c1, "Bool")],
                        blocks=[B.block([], B.s(mu1[b], "Double")), B.block([], B.s(mu0[b], "Double"))])
            row = B.stmt(body, "Times", "Int", [B.i(d), B.s(i2, "Int")])
            ia = row if a == 0 else B.stmt(body, "Plus", "Int", [B.i(a), B.s(row, "Int")])
            xa = B.stmt(body, "VectorApply", "Double", [B.s(x, VD), B.s(ia, "Int")])
            da = B.stmt(body, "Minus", "Double", [B.s(xa, "Double"), B.s(ma, "Double")])
            ib = ia if b == a else row if b == 0 else B.stmt(body, "Plus", "Int", [B.i(b), B.s(row, "Int")])
            xb = B.stmt(body, "VectorApply", "Double", [B.s(x, VD), B.s(ib, "Int")])
            db = B.stmt(body, "Minus", "Double", [B.s(xb, "Double"), B.s(mb, "Double")])
            pr = B.stmt(body, "Times", "Double", [B.s(da, "Double"), B.s(db, "Double")])
            o = B.sym()
            outs.append(o)
            elems.append(B.reduce_elem(o, "Double", B.block(body, B.s(pr, "Double")), -1, B.d(0.0)))
    loop2 = outs[0]
    B.stmts[str(loop2)] = {"op": "ParallelLoop", "ty": "Double", "args": [],
                           "loop": {"range": B.i(n), "index": i2, "body": B.block([], {"u": 1, "t": "Unit"}, bound=[i2]),
                                    "elems": elems}}
    root.append(loop2)
    for o in outs:
        B.stmt(root, "Print", "Unit", [B.s(o, "Double")])
    B.blocks["0"] = {"stmts": root, "result": {"u": 1, "t": "Unit"}, "bound": []}
    return {"format": "dlx-program/1", "root": 0, "stmts": B.stmts, "blocks": B.blocks}


def groupby_program(n: int, K: int) -> dict:
    """The staged program of integration/stage_programs.cpp::groupby(n, K) (pinned statement by
    statement to the reference-staged groupby_n100000_k16 fixture): keys = randIntVector(n, K),
    ONE fused loop of K count reduces predicated on keys(i) == b (vectordsl.cpp:138-151), every
    count printed."""
    B = _Builder()
    root: list[int] = []
    VI = "Vector[Int]"
    keys = B.stmt(root, "VectorRandInt", VI, [B.i(n), B.i(K)])
    i = B.sym()
    outs, elems = [], []
    for b in range(K):
        cb: list[int] = []
        kv = B.stmt(cb, "VectorApply", "Int", [B.s(keys, VI), B.s(i, "Int")])
        q = B.stmt(cb, "Eq", "Bool", [B.s(kv, "Int"), B.i(b)])
        o = B.sym()
        outs.append(o)
        elems.append(B.reduce_elem(o, "Int", B.block([], B.i(1)), B.block(cb, B.s(q, "Bool")), B.i(0)))
    B.stmts[str(outs[0])] = {"op": "ParallelLoop", "ty": "Int", "args": [],
                             "loop": {"range": B.i(n), "index": i, "body": B.block([], {"u": 1, "t": "Unit"}, bound=[i]),
                                      "elems": elems}}
    root.append(outs[0])
    for o in outs:
        B.stmt(root, "Print", "Unit", [B.s(o, "Int")])
    B.blocks["0"] = {"stmts": root, "result": {"u": 1, "t": "Unit"}, "bound": []}
    return {"format": "dlx-program/1", "root": 0, "stmts": B.stmts, "blocks": B.blocks}


def logreg_program(n: int, d: int, iters: int, alpha: float, link: str = "sigmoid") -> dict:
    """The staged program of integration/stage_programs.cpp::logreg(n, d, iters, alpha) in the
    shape the reference's staging + fusion produce (tests/test_descriptors.py compares the softsign
    form statement by statement with the reference-staged logreg_n20000_d8_it2 fixture):
    x = randVector(n*d), y = randIntVector(n, 2), theta = zeros(d); per iteration ONE fused loop of
    a collect h(i) = link(theta . x_i) (printed: h escapes) and d gradient reduces
    (h(i) - toDouble(y(i))) * x(i*d + j), then theta(j) = theta(j) - alpha * g_j on the host;
    theta printed at the end.  link: "softsign" t / (1 + |t|) (the reference has no exp,
    node.hpp:15-27) or "sigmoid" 1 / (1 + exp(0 - t)) (the MathExp extension)."""
    B = _Builder()
    root: list[int] = []
    VD, VI = "Vector[Double]", "Vector[Int]"
    x = B.stmt(root, "VectorRand", VD, [B.i(n * d)])
    y = B.stmt(root, "VectorRandInt", VI, [B.i(n), B.i(2)])
    th = B.stmt(root, "VectorNew", VD, [B.i(d)], aux_ty="Double")
    for _ in range(iters):
        i = B.sym()
        h = B.sym()
        # collect elem: the dot (one nested reduce over j), then the link
        eb: list[int] = []
        j = B.sym()
        dot = B.sym()
        body: list[int] = []
        row = B.stmt(body, "Times", "Int", [B.i(d), B.s(i, "Int")])
        xi = B.stmt(body, "Plus", "Int", [B.s(row, "Int"), B.s(j, "Int")])
        xv = B.stmt(body, "VectorApply", "Double", [B.s(x, VD), B.s(xi, "Int")])
        tv = B.stmt(body, "VectorApply", "Double", [B.s(th, VD), B.s(j, "Int")])
        pr = B.stmt(body, "Times", "Double", [B.s(tv, "Double"), B.s(xv, "Double")])
        inner = B.reduce_elem(dot, "Double", B.block(body, B.s(pr, "Double")), -1, B.d(0.0))
        B.stmts[str(dot)] = {"op": "ParallelLoop", "ty": "Double", "args": [],
                             "loop": {"range": B.i(d), "index": j, "body": B.block([], {"u": 1, "t": "Unit"}, bound=[j]),
                                      "elems": [inner]}}
        eb.append(dot)
        if link == "softsign":
            ab = B.stmt(eb, "MathAbs", "Double", [B.s(dot, "Double")])
            den = B.stmt(eb, "Plus", "Double", [B.d(1.0), B.s(ab, "Double")])
            hv = B.stmt(eb, "Divide", "Double", [B.s(dot, "Double"), B.s(den, "Double")])
        elif link == "sigmoid":
            neg = B.stmt(eb, "Minus", "Double", [B.d(0.0), B.s(dot, "Double")])
            ex = B.stmt(eb, "MathExp", "Double", [B.s(neg, "Double")])
            den = B.stmt(eb, "Plus", "Double", [B.d(1.0), B.s(ex, "Double")])
            hv = B.stmt(eb, "Divide", "Double", [B.d(1.0), B.s(den, "Double")])
        else:
            raise ValueError(link)
        elems = [{"kind": "collect", "live": True, "out": h, "out_ty": VD, "elem": B.block(eb, B.s(hv, "Double")),
                  "cond": -1, "combine": -1, "append": False}]
        grads = []
        for jj in range(d):
            body = []
            row = B.stmt(body, "Times", "Int", [B.i(d), B.s(i, "Int")])
            ix = row if jj == 0 else B.stmt(body, "Plus", "Int", [B.i(jj), B.s(row, "Int")])
            xv = B.stmt(body, "VectorApply", "Double", [B.s(x, VD), B.s(ix, "Int")])
            yv = B.stmt(body, "VectorApply", "Int", [B.s(y, VI), B.s(i, "Int")])
            yd = B.stmt(body, "ToDouble", "Double", [B.s(yv, "Int")])
            r = B.stmt(body, "Minus", "Double", [B.s(hv, "Double"), B.s(yd, "Double")])
            pr = B.stmt(body, "Times", "Double", [B.s(r, "Double"), B.s(xv, "Double")])
            g = B.sym()
            grads.append(g)
            elems.append(B.reduce_elem(g, "Double", B.block(body, B.s(pr, "Double")), -1, B.d(0.0)))
        B.stmts[str(h)] = {"op": "ParallelLoop", "ty": VD, "args": [],
                           "loop": {"range": B.i(n), "index": i, "body": B.block([], {"u": 1, "t": "Unit"}, bound=[i]),
                                    "elems": elems}}
        root.append(h)
        h0 = B.stmt(root, "VectorApply", "Double", [B.s(h, VD), B.i(0)])
        B.stmt(root, "Print", "Unit", [B.s(h0, "Double")])
        for jj in range(d):
            t = B.stmt(root, "Times", "Double", [B.d(alpha), B.s(grads[jj], "Double")])
            a = B.stmt(root, "VectorApply", "Double", [B.s(th, VD), B.i(jj)])
            m = B.stmt(root, "Minus", "Double", [B.s(a, "Double"), B.s(t, "Double")])
            B.stmt(root, "VectorUpdate", "Unit", [B.s(th, VD), B.i(jj), B.s(m, "Double")])
    for jj in range(d):
        v = B.stmt(root, "VectorApply", "Double", [B.s(th, VD), B.i(jj)])
        B.stmt(root, "Print", "Unit", [B.s(v, "Double")])
    B.blocks["0"] = {"stmts": root, "result": {"u": 1, "t": "Unit"}, "bound": []}
    return {"format": "dlx-program/1", "root": 0, "stmts": B.stmts, "blocks": B.blocks}


if __name__ == "__main__":   # python -m paper_1109_0778_b200.descriptors N D K ITERS > out.json
    import sys
    n, d, k, it = (int(v) for v in sys.argv[1:5])
    json.dump({"seed": 1, "program": kmeans_program(n, d, k, it)}, sys.stdout)
