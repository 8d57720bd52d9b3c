set -u
OUT=gpurun_out/r39; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python bench.py --config c4 --steps 30 --warmup 3 --no-cpu-baseline > $OUT/bench_x8.json 2> $OUT/bench_x8.err
F="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
make -s -j8 -C paper_1109_0778_b200 NVFLAGS="$F -DDLX_KMEANS_EPI_PIPE" > $OUT/build_pipe.log 2>&1
timeout 300 python bench.py --config c4 --steps 30 --warmup 3 --no-cpu-baseline > $OUT/bench_pipe.json 2> $OUT/bench_pipe.err
timeout 600 python -m pytest tests -m gpu -q -x -k "screened or c1_step or c4 or kmeans" > $OUT/pytest_pipe.log 2>&1; echo "rc=$?" >> $OUT/pytest_pipe.log
make -s -j8 -C paper_1109_0778_b200 NVFLAGS="$F -DDLX_KMEANS_EPI_PIPE -DDLX_KMEANS_TRACE" > $OUT/build_pipet.log 2>&1
DLX_KMEANS_TRACE=1 timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_trace.json 2> $OUT/trace.err
