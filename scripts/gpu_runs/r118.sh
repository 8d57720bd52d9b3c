#!/bin/bash
# converters' L2 prefetch distance 0/2/3/4 tiles; parity on the default
OUT=gpurun_out/r118; mkdir -p $OUT
F="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
for A in 2 3 4 0 2 3 4 0; do
  make -s -j16 -C paper_1109_0778_b200 NVFLAGS="$F -DDLX_KMEANS_L2_AHEAD=$A" > $OUT/build.log 2>&1
  timeout 300 python bench.py --config c4 --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('ahead=$A', round(r['value'],1), round(r['roofline']['frac'],4))" >> $OUT/res.txt
done
make -s -j16 -C paper_1109_0778_b200 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "screened or c4 or c1 or kmeans" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for c in c4shard8 c4; do timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('default $c', round(r['value'],1), round(r['roofline']['frac'],4))" >> $OUT/res.txt; done
