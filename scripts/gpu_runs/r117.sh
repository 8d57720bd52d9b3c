#!/bin/bash
# converters: L2 bulk prefetch of their rows two tiles ahead (A/B, alternating builds)
OUT=gpurun_out/r117; mkdir -p $OUT
F="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
for V in "-DDLX_KMEANS_L2_AHEAD" "" "-DDLX_KMEANS_L2_AHEAD" "" "-DDLX_KMEANS_L2_AHEAD" ""; do
  make -s -j16 -C paper_1109_0778_b200 NVFLAGS="$F $V" > $OUT/build.log 2>&1
  timeout 300 python bench.py --config c4 --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('variant=[$V]', round(r['value'],1), round(r['roofline']['frac'],4))" >> $OUT/res.txt
done
make -s -j16 -C paper_1109_0778_b200 > /dev/null 2>&1
