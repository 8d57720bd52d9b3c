"""Small invocations of the newer kernels for compute-sanitizer (memcheck / racecheck)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1109_0778_b200 import multiloops as ml  # noqa: E402
from paper_1109_0778_b200.comm import PeerComm  # noqa: E402

x = ml.rng_units(5000 * 16, seed=3).view(5000, 16)
ml.kmeans_step(x, x[:8].clone())                                   # small direct kernel
x3 = ml.rng_units(3001 * 64, seed=4).view(3001, 64)
y3 = ml.rng_ints(3001, 2, seed=4, first_draw=3001 * 64)
ml.gda_fit(x3, y3)                                                 # fused fit + gated fallback
x3b = ml.rng_units(777 * 30, seed=4).view(777, 30)
ml.gda_fit(x3b, ml.rng_ints(777, 2, seed=5))
keys = ml.rng_ints(100_001, 65536, seed=6)
ml.groupby_count(keys, 65536)                                      # 2-CTA cluster histogram
ml.groupby_count(ml.rng_ints(50_001, 131072, seed=7), 131072)      # 4-CTA cluster
c = PeerComm(0, 1, cap_bytes=1 << 20)
cnt = torch.arange(16, dtype=torch.int64, device="cuda")
s = torch.rand(16, 64, dtype=torch.float64, device="cuda")
mu = torch.empty_like(s)
c.kmeans_update_(cnt, s, mu)                                       # peer exchange kernel
c.close()
torch.cuda.synchronize()
print("ok")
