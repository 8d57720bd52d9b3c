#!/bin/bash
# GDA pass 2: centring warps 4/8 x D buffers 2/3
OUT=gpurun_out/r74; mkdir -p $OUT
BASE="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
for V in "4 2" "8 2" "4 3" "8 3" "12 2"; do
  set -- $V
  make -C paper_1109_0778_b200 -j16 NVFLAGS="$BASE -DDLX_GDA_CTR_WARPS=$1 -DDLX_GDA_DBUFS=$2" > $OUT/build_$1_$2.log 2>&1
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "gda_shapes" > $OUT/pytest_$1_$2.log 2>&1; echo "rc=$?" >> $OUT/pytest_$1_$2.log
  timeout 300 python bench.py --config c3 --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('ctr=$1 dbufs=$2', round(r['value'],1), r['ms_per_step'])" >> $OUT/res.txt
done
make -C paper_1109_0778_b200 -j16 > /dev/null 2>&1
