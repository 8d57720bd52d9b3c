#!/bin/bash
# single-pass GDA fit: 8 vs 12 centring warps; parity on the default
OUT=gpurun_out/r81; mkdir -p $OUT
BASE="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
for W in 12 8; do
  make -C paper_1109_0778_b200 -j16 NVFLAGS="$BASE -DDLX_GDA_CTR_WARPS=$W" > $OUT/build_$W.log 2>&1
  timeout 300 python bench.py --config c3 --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('ctr=$W', round(r['value'],1), r['ms_per_step'], round(r['roofline']['frac'],4))" >> $OUT/res.txt
done
make -C paper_1109_0778_b200 -j16 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "gda" > $OUT/pytest_gda.log 2>&1; echo "rc=$?" >> $OUT/pytest_gda.log
