#!/bin/bash
# executor A/B (mirrors on / off), repeated to see the spread
OUT=gpurun_out/r112; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for i in 1 2 3; do timeout 900 python scripts/time_programs.py > $OUT/times_$i.txt 2>&1; done
