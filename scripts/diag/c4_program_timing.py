import sys, time, json, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1109_0778_b200.descriptors import kmeans_program
from paper_1109_0778_b200.program import Program
n, d, k, it = 16777216, 64, 64, int(sys.argv[1])
p = Program(kmeans_program(n, d, k, it))
p.run(seed=1)
for serial in (False, True):
    ts = []
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter(); p.run(seed=1, serial=serial); ts.append((time.perf_counter() - t0) * 1e3)
    print("serial" if serial else "async", [round(t, 2) for t in ts], flush=True)
