#!/bin/bash
# which part of the tail warp slows its SMSP's converter: polling (sleep back-off) or the work (skipped)
OUT=gpurun_out/r123; mkdir -p $OUT
F="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
for V in "" "-DDLX_EXP_TAIL_SLEEP" "-DDLX_EXP_TAIL_NOWORK"; do
  make -s -j16 -C paper_1109_0778_b200 NVFLAGS="$F -DDLX_KMEANS_TRACE -DDLX_TRACE_CONV $V" > $OUT/buildt.log 2>&1
  echo "== [$V]" >> $OUT/trace.txt
  DLX_KMEANS_TRACE=1 timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2> $OUT/t.err
  grep "tile period" $OUT/t.err | head -2 >> $OUT/trace.txt
  make -s -j16 -C paper_1109_0778_b200 NVFLAGS="$F $V" > $OUT/build.log 2>&1
  timeout 300 python bench.py --config c4 --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('variant=[$V]', round(r['value'],1), round(r['roofline']['frac'],4))" >> $OUT/res.txt
done
make -s -j16 -C paper_1109_0778_b200 > /dev/null 2>&1
