set -u
OUT=gpurun_out/r62; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -rf -x -k "screened or c1_step or c4 or kmeans or staged" > $OUT/pytest_k.log 2>&1; echo "rc=$?" >> $OUT/pytest_k.log
for i in 1 2; do
  timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c4_$i.json 2> $OUT/bench_c4_$i.err
done
timeout 300 python bench.py --config c4shard8 --steps 30 --warmup 3 --no-cpu-baseline > $OUT/bench_c4shard8.json 2> $OUT/bench_c4shard8.err
F="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
make -s -j8 -C paper_1109_0778_b200 NVFLAGS="$F -DDLX_KMEANS_TRACE" > $OUT/buildt.log 2>&1
DLX_KMEANS_TRACE=1 timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_trace.json 2> $OUT/trace.err
