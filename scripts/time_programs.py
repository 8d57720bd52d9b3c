"""Wall time of each staged reference program through dlx_program_run (the drop-in executor),
with the host mirrors of small vectors on (default) and off (DLX_PROGRAM_NO_MIRROR=1)."""
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

for path in sorted(glob.glob("tests/golden/staged/*.json")):
    res = {}
    for mode, env in (("mirror", {}), ("per_element", {"DLX_PROGRAM_NO_MIRROR": "1"})):
        out = subprocess.run([sys.executable, __file__, path], env={**os.environ, **env},
                             capture_output=True, text=True)
        res[mode] = float(out.stdout.strip().splitlines()[-1]) if out.returncode == 0 else out.stderr[-200:]
    print(json.dumps({"program": os.path.basename(path)[:-5], "ms": res}), flush=True)
