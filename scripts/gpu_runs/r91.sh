#!/bin/bash
# bench: the step's launches captured in CUDA graphs (launch-bound configs)
OUT=gpurun_out/r91; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for c in c1 c2 c4 c3 c5 l16; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_$c.json 2>$OUT/err_$c
done
