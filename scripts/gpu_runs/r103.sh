#!/bin/bash
# compute-sanitizer on the headline kernels (tcgen05 screened k-means, logreg, GDA pass 1, GroupBy)
OUT=gpurun_out/r103; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 compute-sanitizer --tool memcheck python scripts/diag/sanitize_screened.py > $OUT/memcheck.log 2>&1; echo "rc=$?" >> $OUT/memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard python scripts/diag/sanitize_screened.py > $OUT/racecheck.log 2>&1; echo "rc=$?" >> $OUT/racecheck.log
