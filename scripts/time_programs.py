"""Wall time of each staged reference program through dlx_program_run (the drop-in executor):
default (host mirrors of small vectors, independent loops overlapped on loop streams), with
every loop completed before the next statement (DLX_PROGRAM_SERIAL=1), and with per-element
transfers (DLX_PROGRAM_NO_MIRROR=1).  Also two merged programs whose first loops are
independent (tests/test_staged_programs.py::_merge_independent)."""
import glob
import json
import os
import subprocess
import sys

if len(sys.argv) > 1:   # child: time one fixture
    sys.path.insert(0, ".")
    import time
    from paper_1109_0778_b200.program import run_program
    fx = json.load(open(sys.argv[1]))
    run_program(fx["program"], seed=fx["seed"])            # warm (module load, CUDA context)
    ts = []
    for _ in range(9):
        t0 = time.perf_counter()
        run_program(fx["program"], seed=fx["seed"])
        ts.append((time.perf_counter() - t0) * 1e3)
    print(sorted(ts)[len(ts) // 2])   # median
    sys.exit(0)

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from test_staged_programs import _merge_independent, load  # noqa: E402

paths = sorted(glob.glob("tests/golden/staged/*.json"))
os.makedirs("gpurun_out/merged", exist_ok=True)
for a, b in (("mean_variance_n100000", "groupby_n100000_k16"), ("kmeans_n65536_d16_k8_it1", "gda_n20000_d4")):
    path = f"gpurun_out/merged/{a}+{b}.json"
    with open(path, "w") as f:
        json.dump({"seed": 1, "program": _merge_independent(load(a)["program"], load(b)["program"])}, f)
    paths.append(path)
for path in paths:
    res = {}
    for mode, env in (("overlap", {}), ("serial", {"DLX_PROGRAM_SERIAL": "1"}),
                      ("per_element", {"DLX_PROGRAM_NO_MIRROR": "1"})):
        out = subprocess.run([sys.executable, __file__, path], env={**os.environ, **env},
                             capture_output=True, text=True)
        res[mode] = float(out.stdout.strip().splitlines()[-1]) if out.returncode == 0 else out.stderr[-200:]
    print(json.dumps({"program": os.path.basename(path)[:-5], "ms": res}), flush=True)
