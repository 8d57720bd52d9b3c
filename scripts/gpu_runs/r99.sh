#!/bin/bash
# C1 launch list (per-kernel durations)
OUT=gpurun_out/r99; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches_c1.csv \
  python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/ncu.log 2>&1
