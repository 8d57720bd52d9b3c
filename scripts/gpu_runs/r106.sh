#!/bin/bash
# screened prologue: centroid loads all in flight before the stores; trace phases + bench
OUT=gpurun_out/r106; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "screened or c4 or c1" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for c in c4 c4shard8 c4 c4shard8; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('$c', round(r['value'],1), round(r['roofline']['frac'],4), r['ms_per_step'])" >> $OUT/res.txt
done
F="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
make -s -j16 -C paper_1109_0778_b200 NVFLAGS="$F -DDLX_KMEANS_TRACE" > $OUT/buildt.log 2>&1
DLX_KMEANS_TRACE=1 timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2> $OUT/trace.err
make -s -j16 -C paper_1109_0778_b200 > /dev/null 2>&1
