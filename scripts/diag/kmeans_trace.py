"""Phase / tile-period trace of the screened k-means kernel (a -DDLX_KMEANS_TRACE build loaded
with DLX_LIB_PATH, run with DLX_KMEANS_TRACE=1): 4 iterations at N (default C4), d = k = 64;
the library prints one [dlx phases] / [dlx trace] line per launch to stderr."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1109_0778_b200 import multiloops as ml  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
x = ml.rng_units(n * 64, seed=1).view(n, 64)
mu = x[:64].clone()
a = torch.empty(n, dtype=torch.int32, device="cuda")
c = torch.empty(64, dtype=torch.int64, device="cuda")
s = torch.empty((64, 64), dtype=torch.float64, device="cuda")
for _ in range(4):
    ml.kmeans_step(x, mu, a, c, s, method=2)
    ml.kmeans_update(c, s, mu)
torch.cuda.synchronize()
print("pending", ml.kmeans_last_recheck_count(n, 64, 64))
