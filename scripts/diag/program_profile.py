"""DLX_PROGRAM_PROFILE timeline of one warm run of a BASELINE config's staged program
(stderr): host time of launches / joins and the loops' device intervals.
    DLX_PROGRAM_PROFILE=1 python scripts/diag/program_profile.py c3"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from program_times import CONFIGS, build  # noqa: E402
from paper_1109_0778_b200.program import Program  # noqa: E402

fam, p = CONFIGS[sys.argv[1]]
prog = Program(json.dumps(build(fam, p, p["iters"])))
for _ in range(3):
    print("---- run", file=sys.stderr, flush=True)
    prog.run(seed=1)
