#!/bin/bash
# GroupBy cluster path generalised to 2/4/8-CTA clusters (K up to 400K)
OUT=gpurun_out/r88; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -rf -k "groupby" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for c in c5 c5k4096 c5k65536 c5k262144; do
timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>$OUT/err | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('$c', round(r['value'],1), r['ms_per_step'], round(r['roofline']['frac'],4))" >> $OUT/res.txt
done
