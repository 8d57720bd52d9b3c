"""C4 (k-means N = 16M, d = 64, k = 64, one iteration) as a staged program — built directly in the
reference's fused-loop shape (paper_1109_0778_b200/descriptors.py; the reference's own fusion
pass is quadratic at 4,160 elems), or a descriptor file given as argument (e.g. one staged by
oracle/_ref/stage_programs OUT kmeans_n16777216_d64_k64_it1) — run end to end through the
drop-in executor
(dlx_program_run: one fused loop of 1 collect + 4,160 predicated reduces, recognised as the
k-means family and lowered to the screened tcgen05 kernel; the 4,096 mu updates and 4,161 prints
are host statements).

Checks: the printed assignment of row 0, the 64 counts and the 4,096 updated centroids equal the
family API's result on the same device data bit for bit (ml.kmeans_step, itself bit-exact against
the oracle in tests/test_gpu_parity.py), and the first counts / mu(0) equal SURVEY Appendix B's
C4 iteration-1 goldens.  Prints one JSON line with the executor's wall time per program run.

    python scripts/c4_staged.py [descriptor.json]
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
from paper_1109_0778_b200.program import run_program  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
n, d, k = 16777216, 64, 64
if len(sys.argv) > 1:
    path = sys.argv[1]
    with open(path) as f:
        prog = json.dumps(json.load(f)["program"])
else:
    path = "descriptors.kmeans_program(16777216,64,64,1).json"
    prog = json.dumps(kmeans_program(n, d, k, 1))

t0 = time.perf_counter()
text, report = run_program(prog, seed=1)            # first run: descriptor parse + lowering
first_ms = (time.perf_counter() - t0) * 1e3
ts = []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    text, report = run_program(prog, seed=1)        # parsed descriptor cached by content
    ts.append((time.perf_counter() - t0) * 1e3)
out = [s for s in text.split("\n") if s]
assert len(out) == 1 + k + k * d, len(out)
a0 = int(out[0])
counts = np.array([int(v) for v in out[1:1 + k]], dtype=np.int64)
mu = np.array([float(v) for v in out[1 + k:]], dtype=np.float64).reshape(k, d)

dev = torch.device("cuda", 0)
x = ml.rng_units(n * d, seed=1, device=dev).view(n, d)
torch.cuda.synchronize()
t0 = time.perf_counter()
assign, cnt, sums = ml.kmeans_step(x, x[:k].clone())
torch.cuda.synchronize()
family_ms = (time.perf_counter() - t0) * 1e3
cnt_h = cnt.cpu().numpy()
mu_f = (sums / cnt.to(torch.float64).unsqueeze(1)).cpu().numpy()
ok_assign = a0 == int(assign[0].item())
ok_counts = bool(np.array_equal(counts, cnt_h))
ok_mu = bool(np.array_equal(mu.view(np.int64), mu_f.view(np.int64)))

with open(os.path.join(ROOT, "tests", "golden", "appendix_b.json")) as f:
    g = json.load(f)["c4_kmeans"]
ok_golden = bool([int(v) for v in counts[:4]] == g["counts_prefix"][0]
             and abs(mu[0, 0] - float(g["mu00"][0])) <= 1e-9 * abs(float(g["mu00"][0])))

# the same program without its loop (x drawn, mu initialised and printed): the executor's
# host-statement and allocation share of a run
prog0 = json.dumps(kmeans_program(n, d, k, 0))
run_program(prog0, seed=1)
t0s = []
for _ in range(3):
    t0 = time.perf_counter()
    run_program(prog0, seed=1)
    t0s.append((time.perf_counter() - t0) * 1e3)

loop = [r for r in report if r.get("launch")]
print(json.dumps({
    "program": os.path.basename(path)[:-5], "descriptor_mb": round(len(prog) / 2**20, 1),
    "live_elems": loop[0]["live_elems"] if loop else None, "family": [r["family"] for r in report],
    "first_run_ms": round(first_ms, 1), "run_ms_median": round(sorted(ts)[len(ts) // 2], 2),
    "run_ms": [round(t, 2) for t in ts], "no_loop_run_ms": round(sorted(t0s)[1], 2),
    "family_api_step_ms": round(family_ms, 2), "pool_keep_gb": os.environ.get("DLX_POOL_KEEP_GB", "32 (default)"),
    "match_family_api": {"assign0": ok_assign, "counts": ok_counts, "mu_bits": ok_mu},
    "appendix_b": ok_golden}))
assert ok_assign and ok_counts and ok_mu and ok_golden
