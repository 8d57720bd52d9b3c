"""C4 (k-means N = 16M, d = 64, k = 64) as a staged program of ITERS fused iterations, built in the
reference's fused-loop shape (paper_1109_0778_b200/descriptors.py; tests/test_descriptors.py pins
the builder statement by statement against the reference-staged fixtures) — or a descriptor
file given as argument — run end to end through the drop-in executor (dlx_program_create once,
dlx_program_execute per run: x drawn on the device, mu initialised from x's first rows by k*d
host statements, ITERS fused loops of 1 collect + 4,160 predicated reduces lowered to the
screened tcgen05 kernel with the k*d centroid updates on the device, 65 prints per iteration,
the k*d final centroids printed).

Checks: the printed assignment of row 0 and counts of every iteration and the final centroids
equal the family API's iterations on the same device data bit for bit, and iteration 1's
counts prefix / mu(0) equal SURVEY Appendix B.  Prints one JSON line: wall time per program
run, per iteration, and the same program without its loops.

    python scripts/c4_staged.py [ITERS] [descriptor.json]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1109_0778_b200 import multiloops as ml  # noqa: E402
from paper_1109_0778_b200.descriptors import kmeans_program  # noqa: E402
from paper_1109_0778_b200.program import Program  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
n, d, k = 16777216, 64, 64
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 10
if len(sys.argv) > 2:
    with open(sys.argv[2]) as f:
        desc = json.load(f)["program"]
    name = os.path.basename(sys.argv[2])[:-5]
else:
    desc = kmeans_program(n, d, k, iters)
    name = f"descriptors.kmeans_program({n},{d},{k},{iters})"
text_desc = json.dumps(desc)
t0 = time.perf_counter()
prog = Program(text_desc)
create_ms = (time.perf_counter() - t0) * 1e3
t0 = time.perf_counter()
r = prog.run(seed=1)                                 # first run: lowers every loop
first_ms = (time.perf_counter() - t0) * 1e3
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = prog.run(seed=1)                             # lowerings cached in the handle
    ts.append((time.perf_counter() - t0) * 1e3)
out = [s for s in r.output.split("\n") if s]
per = 1 + k
assert len(out) == iters * per + k * d, len(out)

dev = torch.device("cuda", 0)
x = ml.rng_units(n * d, seed=1, device=dev).view(n, d)
mu = x[:k].clone()
ok_assign = ok_counts = True
counts_it = []
torch.cuda.synchronize()
t0 = time.perf_counter()
for t in range(iters):
    a, c, s = ml.kmeans_step(x, mu)
    ok_assign &= int(out[t * per]) == int(a[0].item())
    ch = c.cpu().numpy()
    counts_it.append(ch)
    ok_counts &= [int(v) for v in out[t * per + 1:(t + 1) * per]] == ch.tolist()
    mu = ml.kmeans_update(c, s)
torch.cuda.synchronize()
family_ms = (time.perf_counter() - t0) * 1e3
mu_p = np.array([float(v) for v in out[iters * per:]])
ok_mu = bool(np.array_equal(mu_p.view(np.int64), mu.cpu().numpy().reshape(-1).view(np.int64)))
with open(os.path.join(ROOT, "tests", "golden", "appendix_b.json")) as f:
    g = json.load(f)["c4_kmeans"]
ok_golden = [int(v) for v in counts_it[0][:4]] == g["counts_prefix"][0]
del x

# the same program without its loops (x drawn, mu initialised and printed): the executor's
# host-statement and allocation share of a run
prog0 = Program(kmeans_program(n, d, k, 0))
prog0.run(seed=1)
t0s = []
for _ in range(3):
    t0 = time.perf_counter()
    prog0.run(seed=1)
    t0s.append((time.perf_counter() - t0) * 1e3)
med = sorted(ts)[len(ts) // 2]
no_loop = sorted(t0s)[1]
print(json.dumps({
    "program": name, "iterations": iters, "descriptor_mb": round(len(text_desc) / 2**20, 1),
    "live_elems": r.report[0]["live_elems"], "family": sorted({e["family"] for e in r.report}),
    "update": sorted({e.get("update", "") for e in r.report}), "cached": all(e["cached"] for e in r.report),
    "create_ms": round(create_ms, 1), "first_run_ms": round(first_ms, 1), "run_ms_median": round(med, 2),
    "run_ms": [round(t, 2) for t in ts], "ms_per_iteration": round(med / iters, 3),
    "no_loop_run_ms": round(no_loop, 2), "ms_per_iteration_marginal": round((med - no_loop) / iters, 3),
    "family_api_ms_per_iteration": round(family_ms / iters, 3),
    "match_family_api": {"assign0": ok_assign, "counts": ok_counts, "mu_bits": ok_mu}, "appendix_b": ok_golden}))
assert ok_assign and ok_counts and ok_mu and ok_golden
