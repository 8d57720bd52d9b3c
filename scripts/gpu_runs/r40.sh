set -u
OUT=gpurun_out/r40; mkdir -p $OUT
F="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
make -s -j8 -C paper_1109_0778_b200 NVFLAGS="$F -DDLX_KMEANS_DIAG_NOFOLD -DDLX_KMEANS_TRACE" > $OUT/build.log 2>&1
DLX_KMEANS_TRACE=1 timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_trace.json 2> $OUT/trace.err
make -s -j8 -C paper_1109_0778_b200 NVFLAGS="$F -DDLX_KMEANS_DIAG_NOFOLD" > $OUT/build2.log 2>&1
timeout 300 python bench.py --config c4 --steps 30 --warmup 3 --no-cpu-baseline > $OUT/bench_nofold.json 2> $OUT/bench_nofold.err
