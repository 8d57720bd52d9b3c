#!/bin/bash
# k-means iteration with the centroid update fused into the combine launch: tests + A/B
OUT=gpurun_out/r138; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
for rep in 1 2; do for V in 0 1; do for c in c1 c4shard8 c4; do
  DLX_KMEANS_UNFUSED_UPDATE=$V timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('$c unfused=$V', round(r['value'],1), round(r['roofline']['frac'],4), r['gpu_launches'])" >> $OUT/res.txt
done; done; done
