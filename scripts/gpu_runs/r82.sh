#!/bin/bash
# c4shard8 (2M-row shard): launch list and per-phase trace of the screened kernel
OUT=gpurun_out/r82; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python bench.py --config c4shard8 --steps 30 --warmup 5 --no-cpu-baseline > $OUT/bench_c4shard8.json 2> $OUT/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches.csv \
  python bench.py --config c4shard8 --steps 4 --warmup 3 --no-cpu-baseline > $OUT/ncu2.log 2>&1
