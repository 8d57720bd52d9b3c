#!/bin/bash
# screen MMAs per tile: 8 (default) vs 7 (DLX_KMEANS_SCREEN7=1), alternating builds
OUT=gpurun_out/r126; mkdir -p $OUT
F="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
for V in 0 1 0 1 0 1; do
  make -s -j16 -C paper_1109_0778_b200 NVFLAGS="$F -DDLX_KMEANS_SCREEN7=$V" > $OUT/build.log 2>&1
  timeout 300 python bench.py --config c4 --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('screen7=$V', round(r['value'],1), round(r['roofline']['frac'],4))" >> $OUT/res.txt
done
make -s -j16 -C paper_1109_0778_b200 > /dev/null 2>&1
