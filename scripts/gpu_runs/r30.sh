set -u
OUT=gpurun_out/r30; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c16.json 2> $OUT/bench_c16.err
F="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
make -s -B -j8 -C paper_1109_0778_b200 NVFLAGS="$F -DDLX_KMEANS_CONV_WARPS=8" > $OUT/build8.log 2>&1
timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c8.json 2> $OUT/bench_c8.err
timeout 600 python -m pytest tests -m gpu -q -x -k "screened or c1_step or c4 or kmeans" > $OUT/pytest_c8.log 2>&1
make -s -B -j8 -C paper_1109_0778_b200 NVFLAGS="$F -DDLX_KMEANS_CONV_WARPS=8 -DDLX_KMEANS_TRACE" > $OUT/build8t.log 2>&1
DLX_KMEANS_TRACE=1 timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_trace8.json 2> $OUT/trace8.err
