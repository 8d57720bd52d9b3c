"""Generate tests/golden/oracle_hashes.json: fnv64w hashes of assignments / counts computed by
the CPU oracle (sequential interpret order, chunks=1) at the SURVEY App. B configs.

These complement appendix_b.json: the counts, centroids and SHA-256 texts there are matched
exactly by the oracle (tests/test_oracle.py), which pins the oracle; the App. B fnv64w values
themselves do not reproduce under their stated definition, so the hashes used by the GPU parity
tests are regenerated here from the pinned oracle.

    python tests/golden/make_oracle_hashes.py          # ~2 minutes, 10 GB RAM
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import oracle as O  # noqa: E402


def main():
    out = {"_source": "oracle (sequential, chunks=1) — see make_oracle_hashes.py"}
    x, mu0 = O.kmeans_inputs(65536, 16, 8)
    hist = O.kmeans_run(x, 8, 10, mu0)
    out["c1_assign_fnv64w"] = [hex(h[1]) for h in hist]
    out["c1_counts_fnv64w"] = [hex(O.fnv64w(h[0])) for h in hist]
    del x
    x, mu = O.kmeans_inputs(16777216, 64, 64)
    c4a, c4c = [], []
    for it in range(2):
        a, c, s = O.kmeans_step(x, 64, mu, workers=1, chunks=1)
        c4a.append(hex(O.fnv64w(a)))
        c4c.append(hex(O.fnv64w(c)))
        mu = O.kmeans_update(c, s)
        print("c4 iteration", it + 1, c[:4].tolist(), O.format_double(s[0, 0]), O.format_double(mu[0, 0]), flush=True)
    out["c4_assign_fnv64w"] = c4a
    out["c4_counts_fnv64w"] = c4c
    del x
    n = 10 ** 9
    out["c5_counts_fnv64w"] = {}
    for K in (64, 4096, 65536):
        keys = O.rng_ints(1, 0, n, K)
        out["c5_counts_fnv64w"][str(K)] = hex(O.fnv64w(O.groupby_count(keys, K, workers=O.threads(), chunks=4 * O.threads())))
        del keys
    path = os.path.join(os.path.dirname(__file__), "oracle_hashes.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
