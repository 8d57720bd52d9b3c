#!/bin/bash
# compute-sanitizer memcheck + racecheck on small invocations of the newer kernels
OUT=gpurun_out/r102; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 compute-sanitizer --tool memcheck python scripts/diag/sanitize_small.py > $OUT/memcheck.log 2>&1; echo "rc=$?" >> $OUT/memcheck.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python scripts/diag/sanitize_small.py > $OUT/racecheck.log 2>&1; echo "rc=$?" >> $OUT/racecheck.log
timeout 900 compute-sanitizer --tool initcheck python scripts/diag/sanitize_small.py > $OUT/initcheck.log 2>&1; echo "rc=$?" >> $OUT/initcheck.log
