#!/bin/bash
# k-means method crossover: direct fp64 vs tcgen05 screened at small N
OUT=gpurun_out/r83; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for m in 1 2; do
  timeout 300 python bench.py --config c1 --steps 200 --warmup 10 --method $m --no-cpu-baseline 2>/dev/null | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('c1 method=$m', round(r['value'],1), r['ms_per_step'], r['roofline']['kernel_ms'])" >> $OUT/res.txt
done
timeout 900 python scripts/kmeans_crossover.py > $OUT/crossover.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
