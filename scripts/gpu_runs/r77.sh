#!/bin/bash
# logreg: row-kernel grid multiple x min blocks per SM (occupancy / wave quantisation)
OUT=gpurun_out/r77; mkdir -p $OUT
BASE="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
for V in "4 1" "3 1" "4 4" "8 4" "2 2" "6 3"; do
  set -- $V
  make -C paper_1109_0778_b200 -j16 NVFLAGS="$BASE -DDLX_ROW_GRID_MULT=$1 -DDLX_ROW_MINB=$2" > $OUT/build_$1_$2.log 2>&1
  grep -A2 "logreg_grad_kernelILi1" paper_1109_0778_b200/build/rows.ptxas.log | grep Used >> $OUT/res.txt
  for c in c2 l16; do
    timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('mult=$1 minb=$2 $c', round(r['value'],1), round(r['roofline']['frac'],4), r['roofline']['kernel_ms'])" >> $OUT/res.txt
  done
done
make -C paper_1109_0778_b200 -j16 > /dev/null 2>&1
