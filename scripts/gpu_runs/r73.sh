#!/bin/bash
OUT=gpurun_out/r73; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gda_pass2 -s 2 -c 1 -o $OUT/prof_gda \
  python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu.log 2>&1
