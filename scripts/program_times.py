"""Every BASELINE config as a staged program through the drop-in executor (dlx_program_create
once, dlx_program_execute per run; descriptors built in the reference-staged shape by
paper_1109_0778_b200/descriptors.py), against the family API (multiloops.*) doing the same
iterations on the same device data.  One JSON line per config: median wall ms per program run,
per iteration, the program without its loops (host statements, draws, prints), and the
family API's ms per iteration.

    python scripts/program_times.py [c1 c2 c3 c4 c5]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1109_0778_b200 import descriptors as D  # noqa: E402
from paper_1109_0778_b200 import multiloops as ml  # noqa: E402
from paper_1109_0778_b200.program import Program  # noqa: E402

CONFIGS = {
    "c1": ("kmeans", dict(n=65536, d=16, k=8, iters=10)),
    "c2": ("logreg", dict(n=1 << 20, d=64, iters=20)),
    "c3": ("gda", dict(n=1 << 20, d=64, iters=1)),
    "c4": ("kmeans", dict(n=1 << 24, d=64, k=64, iters=10)),
    "c5": ("groupby", dict(n=10 ** 9, K=64, iters=1)),
}


def build(fam, p, iters):
    if fam == "kmeans":
        return D.kmeans_program(p["n"], p["d"], p["k"], iters)
    if fam == "logreg":
        return D.logreg_program(p["n"], p["d"], iters, 1.0 / p["n"])
    if fam == "gda":
        return D.gda_program(p["n"], p["d"]) if iters else None
    return D.groupby_program(p["n"], p["K"]) if iters else None


def timed(fn, reps):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return sorted(ts)[len(ts) // 2], ts


def family_ms(fam, p):
    dev = torch.device("cuda", 0)
    n = p["n"]
    if fam == "kmeans":
        x = ml.rng_units(n * p["d"], seed=1, device=dev).view(n, p["d"])
        mu = [x[:p["k"]].clone()]

        def it():
            a, c, s = ml.kmeans_step(x, mu[0])
            mu[0] = ml.kmeans_update(c, s)
    elif fam == "logreg":
        x = ml.rng_units(n * p["d"], seed=1, device=dev).view(n, p["d"])
        y = ml.rng_ints(n, 2, seed=1, first_draw=n * p["d"], device=dev)
        th = torch.zeros(p["d"], dtype=torch.float64, device=dev)

        def it():
            g = ml.logreg_grad(x, y, th)
            ml.axpy_inplace(th, g, 1.0 / n)
    elif fam == "gda":
        x = ml.rng_units(n * p["d"], seed=1, device=dev).view(n, p["d"])
        y = ml.rng_ints(n, 2, seed=1, first_draw=n * p["d"], device=dev)

        def it():
            ml.gda_fit(x, y)
    else:
        keys = ml.rng_ints(n, p["K"], seed=1, device=dev)

        def it():
            ml.groupby_count(keys, p["K"])
    it()
    med, _ = timed(lambda: [it() for _ in range(p["iters"])], 5)
    return med / p["iters"]


def main():
    names = sys.argv[1:] or list(CONFIGS)
    for name in names:
        fam, p = CONFIGS[name]
        desc = json.dumps(build(fam, p, p["iters"]))
        t0 = time.perf_counter()
        prog = Program(desc)
        create_ms = (time.perf_counter() - t0) * 1e3
        t0 = time.perf_counter()
        r = prog.run(seed=1)
        first_ms = (time.perf_counter() - t0) * 1e3
        med, ts = timed(lambda: prog.run(seed=1), 7)
        res = {"config": name, "family": sorted({e["family"] for e in r.report}),
               "loops_per_run": len(r.report), "iterations": p["iters"], "descriptor_kb": round(len(desc) / 1024, 1),
               "create_ms": round(create_ms, 1), "first_run_ms": round(first_ms, 1),
               "run_ms_median": round(med, 3), "run_ms": [round(t, 3) for t in ts],
               "ms_per_iteration": round(med / p["iters"], 4)}
        prog.close()
        del prog
        torch.cuda.empty_cache()
        res["family_api_ms_per_iteration"] = round(family_ms(fam, p), 4)
        res["dropin_over_family"] = round(res["ms_per_iteration"] / res["family_api_ms_per_iteration"], 2)
        print(json.dumps(res), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
