"""Per-iteration k-means time vs N (d = 64, k = 64) on one GPU: the fixed per-launch cost
(prologue, pipeline ramp and drain, flush, combine, update) against the per-sample slope."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1109_0778_b200 import multiloops as ml  # noqa: E402


def time_n(n, iters=20):
    x = ml.rng_units(n * 64, seed=1).view(n, 64)
    mu = x[:64].clone()
    a = torch.empty(n, dtype=torch.int32, device="cuda")
    c = torch.empty(64, dtype=torch.int64, device="cuda")
    s = torch.empty((64, 64), dtype=torch.float64, device="cuda")
    for _ in range(3):
        ml.kmeans_step(x, mu, a, c, s)
        ml.kmeans_update(c, s, mu)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        ml.kmeans_step(x, mu, a, c, s)
        ml.kmeans_update(c, s, mu)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


out = {}
for n in (148 * 128, 4 * 148 * 128, 16 * 148 * 128, 1 << 21, 1 << 22, 1 << 24):
    out[n] = time_n(n)
    print(json.dumps({"n": n, "ms_per_iter": out[n]}), flush=True)
