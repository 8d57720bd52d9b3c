#!/bin/bash
# converged MMA/fold issuer warps: per-SMSP converter completion (trace) + A/B bench vs HEAD + parity
OUT=gpurun_out/r124; mkdir -p $OUT
F="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "screened or c4 or c1 or kmeans" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for i in 1 2 3; do
  timeout 300 python bench.py --config c4 --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('new', round(r['value'],1), round(r['roofline']['frac'],4))" >> $OUT/res.txt
done
make -s -j16 -C paper_1109_0778_b200 NVFLAGS="$F -DDLX_KMEANS_TRACE" > $OUT/buildt.log 2>&1
DLX_KMEANS_TRACE=1 timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2> $OUT/trace.err
make -s -j16 -C paper_1109_0778_b200 > /dev/null 2>&1
