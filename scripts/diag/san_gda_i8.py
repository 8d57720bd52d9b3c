import sys, torch
sys.path.insert(0, '.')
from paper_1109_0778_b200 import multiloops as ml
for n in (20_000, 96 * 148 * 2 + 37):
    x = ml.rng_units(n * 64, seed=3).view(n, 64)
    y = ml.rng_ints(n, 2, seed=3, first_draw=n * 64)
    assert ml.gda_fit_path(x, y) in ("int8", "dmma")
    r = ml.gda_fit(x, y)
    torch.cuda.synchronize()
    print("fit ok", n, int(r[0].item()), ml.gda_fit_last_fallback(x))
x[5000, 3] = float("inf")
r = ml.gda_fit(x, y); torch.cuda.synchronize(); print("fallback", ml.gda_fit_last_fallback(x))
