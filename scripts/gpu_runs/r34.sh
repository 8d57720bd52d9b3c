set -u
OUT=gpurun_out/r34; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "screened or c1_step or c4 or kmeans or staged or filter" > $OUT/pytest_k.log 2>&1; echo "rc=$?" >> $OUT/pytest_k.log
timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_s256.json 2> $OUT/bench_s256.err
F="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
for ns in 64 1024; do
  make -s -B -j8 -C paper_1109_0778_b200 NVFLAGS="$F -DDLX_KMEANS_CONV_SLEEP=$ns" > $OUT/build_$ns.log 2>&1
  timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_s$ns.json 2> $OUT/bench_s$ns.err
done
make -s -B -j8 -C paper_1109_0778_b200 NVFLAGS="$F -DDLX_KMEANS_TRACE" > $OUT/build_t.log 2>&1
DLX_KMEANS_TRACE=1 timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_trace.json 2> $OUT/trace.err
