# small screened k-means steps (several tiles per CTA, pending rows) for compute-sanitizer runs
import sys, torch
sys.path.insert(0, '.')
from paper_1109_0778_b200 import multiloops as ml
for n, k in ((40_000, 64), (128 * 148 * 3 + 77, 32)):
    x = ml.rng_units(n * 64, seed=5).view(n, 64)
    mu = x[:k].clone()
    a, c, s = ml.kmeans_step(x, mu, method=2)
    torch.cuda.synchronize()
    print("screened ok", n, k, int(c.sum().item()))
