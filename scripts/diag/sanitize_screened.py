"""Small invocations of the headline kernels for compute-sanitizer."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1109_0778_b200 import multiloops as ml  # noqa: E402

x = ml.rng_units(20_000 * 64, seed=1).view(20_000, 64)
a, c, s = ml.kmeans_step(x, x[:64].clone(), method=2)               # tcgen05 screened <64, true>
x2 = ml.rng_units(3001 * 34, seed=2).view(3001, 34)
ml.kmeans_step(x2, x2[:17].clone(), method=2)                       # generic screened
y = ml.rng_ints(20_000, 2, seed=1)
ml.logreg_grad(x, y, torch.zeros(64, dtype=torch.float64, device="cuda"))
ml.gda_pass1(x, y)
ml.groupby_count(ml.rng_ints(100_000, 64, seed=3), 64)
torch.cuda.synchronize()
print("ok", int(c.sum()))
