"""Per-job wall time of the staged k-means program through dlx_program_execute with the sample
matrix from pinned host memory (bench.py e2e leg), one thread, for a given shape; then one run
under DLX_PROGRAM_PROFILE (stderr).   python scripts/diag/e2e_dropin_profile.py N D K [ITERS]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1109_0778_b200 import multiloops as ml  # noqa: E402
from paper_1109_0778_b200.descriptors import kmeans_program  # noqa: E402
from paper_1109_0778_b200.program import Program  # noqa: E402

n, d, k = (int(v) for v in sys.argv[1:4])
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 10
dev = torch.device("cuda", 0)
desc = kmeans_program(n, d, k, iters)
xsym = next(int(q) for q, st in desc["stmts"].items() if st["op"] == "VectorRand")
x_host = torch.empty(n * d, dtype=torch.float64, pin_memory=True)
x_host.copy_(ml.rng_units(n * d, seed=1, device=dev))
x_dev = ml.rng_units(n * d, seed=1, device=dev)
torch.cuda.synchronize()
prog = Program(desc)
res = {}
for name, inputs in (("generated", None), ("host_input", {xsym: x_host}), ("device_input", {xsym: x_dev})):
    prog.run(seed=1, inputs=inputs)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        prog.run(seed=1, inputs=inputs)
        ts.append((time.perf_counter() - t0) * 1e3)
    res[name] = sorted(ts)[2]
t0 = time.perf_counter()
torch.cuda.synchronize()
h2d = torch.empty(n * d, dtype=torch.float64, device=dev)
torch.cuda.synchronize()
t0 = time.perf_counter()
h2d.copy_(x_host, non_blocking=True)
torch.cuda.synchronize()
res["torch_h2d_ms"] = (time.perf_counter() - t0) * 1e3
print(json.dumps({"n": n, "d": d, "k": k, "iters": iters, "run_ms_median": res}))
os.environ["DLX_PROGRAM_PROFILE"] = "1"
print("---- profiled host-input run", file=sys.stderr, flush=True)
prog.run(seed=1, inputs={xsym: x_host})

# two handles on two host threads (bench.py's e2e form): per-job start / end times
import threading  # noqa: E402
os.environ.pop("DLX_PROGRAM_PROFILE", None)
progs = [prog, Program(desc)]
progs[1].run(seed=1, inputs={xsym: x_host})
marks = []
lock = threading.Lock()
t_base = time.perf_counter()


def worker(t):
    torch.cuda.set_device(dev)
    for j in range(2):
        a = time.perf_counter()
        progs[t].run(seed=1, inputs={xsym: x_host})
        b = time.perf_counter()
        with lock:
            marks.append((t, j, round((a - t_base) * 1e3, 2), round((b - t_base) * 1e3, 2)))


torch.cuda.synchronize()
t_base = time.perf_counter()
ths = [threading.Thread(target=worker, args=(t,)) for t in range(2)]
for th in ths:
    th.start()
for th in ths:
    th.join()
torch.cuda.synchronize()
print(json.dumps({"two_threads_ms": round((time.perf_counter() - t_base) * 1e3, 2), "jobs": sorted(marks)}))
