#!/bin/bash
# GroupBy: max cluster size 2 / 4 / 8 at K = 131072 and 262144 (vs global atomics)
OUT=gpurun_out/r89; mkdir -p $OUT
BASE="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
for C in 2 4 8; do
  make -C paper_1109_0778_b200 -j16 NVFLAGS="$BASE -DDLX_GB_MAX_CLUSTER=$C" > $OUT/build_$C.log 2>&1
  for c in c5k131072 c5k262144; do
    timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>$OUT/err | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('maxC=$C $c', round(r['value'],1), r['ms_per_step'], round(r['roofline']['frac'],4))" >> $OUT/res.txt
  done
done
make -C paper_1109_0778_b200 -j16 > /dev/null 2>&1
