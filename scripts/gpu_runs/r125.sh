#!/bin/bash
# screen: 7 MMAs per tile (the second k-step's h'' products in one N=192 MMA); parity + bench
OUT=gpurun_out/r125; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "screened or c4 or c1 or kmeans" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for i in 1 2 3; do
  timeout 300 python bench.py --config c4 --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('new', round(r['value'],1), round(r['roofline']['frac'],4))" >> $OUT/res.txt
done
