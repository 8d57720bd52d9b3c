#!/bin/bash
# epilogue survivor mask: 2 / 4 / 8 independent funnel-shift chains
OUT=gpurun_out/r97; mkdir -p $OUT
F="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
for C in 8 4 2 8; do
  make -s -j16 -C paper_1109_0778_b200 NVFLAGS="$F -DDLX_KMEANS_MASK_CHAINS=$C" > $OUT/build_$C.log 2>&1
  timeout 300 python bench.py --config c4 --steps 30 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('chains=$C', round(r['value'],1), round(r['roofline']['frac'],4), r['roofline']['kernel_ms'])" >> $OUT/res.txt
done
make -s -j16 -C paper_1109_0778_b200 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "screened or c4 or c1 or kmeans" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
