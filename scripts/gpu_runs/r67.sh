#!/bin/bash
# L2 prefetch of each CTA's first tiles before pdl_wait: 0 / 3 / 6 tiles, c4 and the 2M shard
OUT=gpurun_out/r67; mkdir -p $OUT
BASE="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
for P in 0 3 6 3 0; do
  make -C paper_1109_0778_b200 -j16 NVFLAGS="$BASE -DDLX_KMEANS_PREFETCH_TILES=$P" > $OUT/build_$P.log 2>&1
  for c in c4 c4shard8; do
    timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('P=$P', '$c', round(r['value'],1), round(r['roofline']['frac'],4), r['roofline']['kernel_ms'])" >> $OUT/res.txt
  done
done
make -C paper_1109_0778_b200 -j16 > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "screened or c4" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
