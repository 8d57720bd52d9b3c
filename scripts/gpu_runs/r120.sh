#!/bin/bash
# per-tile trace after the one-hot and L2-prefetch changes
OUT=gpurun_out/r120; mkdir -p $OUT
F="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
make -s -j16 -C paper_1109_0778_b200 NVFLAGS="$F -DDLX_KMEANS_TRACE" > $OUT/buildt.log 2>&1
DLX_KMEANS_TRACE=1 timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2> $OUT/trace.err
make -s -j16 -C paper_1109_0778_b200 > /dev/null 2>&1
