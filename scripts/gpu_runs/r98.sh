#!/bin/bash
# e2e with double-buffered jobs (H2D of job j+1 overlaps job j)
OUT=gpurun_out/r98; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for c in c4 l16 c2 c1; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_$c.json 2>$OUT/err_$c
done
