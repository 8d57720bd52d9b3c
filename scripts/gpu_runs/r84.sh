#!/bin/bash
# GroupBy K sweep (64 / 4096 / 65536)
OUT=gpurun_out/r84; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for c in c5 c5k4096 c5k65536; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>$OUT/$c.err | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('$c', round(r['value'],1), r['ms_per_step'], round(r['roofline']['frac'],4))" >> $OUT/res.txt
done
