#!/bin/bash
# experiment: how fast would the tile loop run if the screen did not wait for the TMEM drain?
OUT=gpurun_out/r96; mkdir -p $OUT
F="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
make -s -j16 -C paper_1109_0778_b200 NVFLAGS="$F -DDLX_KMEANS_TRACE" > $OUT/buildt.log 2>&1
DLX_KMEANS_TRACE=1 timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/base.json 2> $OUT/base.err
make -s -j16 -C paper_1109_0778_b200 NVFLAGS="$F -DDLX_KMEANS_TRACE -DDLX_EXP_EARLY_TEMPTY" > $OUT/buildt2.log 2>&1
DLX_KMEANS_TRACE=1 timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/exp.json 2> $OUT/exp.err
make -s -j16 -C paper_1109_0778_b200 > /dev/null 2>&1
