#!/bin/bash
# row kernels (logreg, GDA pass 1): one full wave, 2 or 3 CTAs per SM
OUT=gpurun_out/r78; mkdir -p $OUT
BASE="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
for V in "2 2" "3 3"; do
  set -- $V
  make -C paper_1109_0778_b200 -j16 NVFLAGS="$BASE -DDLX_ROW_GRID_MULT=$1 -DDLX_ROW_MINB=$2" > $OUT/build_$1_$2.log 2>&1
  grep -A2 "logreg_grad_kernelILi1\|gda_pass1_kernelILi1" paper_1109_0778_b200/build/rows.ptxas.log | grep Used >> $OUT/res.txt
  for c in c2 l16 c3; do
    timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('mult=$1 minb=$2 $c', round(r['value'],1), round(r['roofline']['frac'],4), r['roofline']['kernel_ms'], r.get('roofline_pass1',{}).get('frac'))" >> $OUT/res.txt
  done
done
make -C paper_1109_0778_b200 -j16 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "logreg or gda or c2" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
