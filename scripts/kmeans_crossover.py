"""Per-iteration k-means time, direct fp64 kernel (method 1) vs tcgen05 screened (method 2),
over N for the C1 shape (d = 16, k = 8) and the C4 shape (d = 64, k = 64): where AUTO should
switch."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1109_0778_b200 import multiloops as ml  # noqa: E402


def time_n(n, d, k, method, iters=30):
    x = ml.rng_units(n * d, seed=1).view(n, d)
    mu = x[:k].clone()
    a = torch.empty(n, dtype=torch.int32, device="cuda")
    c = torch.empty(k, dtype=torch.int64, device="cuda")
    s = torch.empty((k, d), dtype=torch.float64, device="cuda")
    for _ in range(3):
        ml.kmeans_step(x, mu, a, c, s, method=method)
        ml.kmeans_update(c, s, mu)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        ml.kmeans_step(x, mu, a, c, s, method=method)
        ml.kmeans_update(c, s, mu)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


for d, k in ((16, 8), (64, 64), (64, 8), (16, 64)):
    for n in (4096, 65536, 262144, 1 << 20, 1 << 22):
        r = {m: time_n(n, d, k, m) for m in (0, 1, 2)}
        print(json.dumps({"d": d, "k": k, "n": n, "auto_ms": r[0], "direct_ms": r[1], "screened_ms": r[2]}), flush=True)
