#!/bin/bash
# C1 launch list (per-kernel time of one graph-replayed step)
OUT=gpurun_out/r137; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 60 --csv --log-file $OUT/launches_c1.csv python bench.py --config c1 --steps 4 --warmup 3 --no-cpu-baseline > $OUT/ncu_c1.log 2>&1
