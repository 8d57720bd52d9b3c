# r319: end-of-launch re-check: all gather loads in flight, the fold by centroid segments in list
# order (register accumulation); A/B vs the committed kernel, phase trace, k-means tests
OUT=gpurun_out/r319; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_program.py tests/test_staged_programs.py -m gpu -q -rf -x --timeout 300 -k "kmeans or screened or c4 or c1" > $OUT/pytest_kmeans.log 2>&1; echo "rc=$?" >> $OUT/pytest_kmeans.log
for n in 16777216 2097152; do
  DLX_LIB_PATH=paper_1109_0778_b200/build_trace/libdlx.so DLX_KMEANS_TRACE=1 timeout 300 python scripts/diag/kmeans_trace.py $n > $OUT/trace_$n.txt 2>&1
done
for i in 1 2 3; do
for v in acc3 new; do
  if [ $v = new ]; then L=""; else L=paper_1109_0778_b200/build_$v/libdlx.so; fi
  for c in c4 c4shard8; do
    DLX_LIB_PATH=$L timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_${c}_${v}_$i.json 2>> $OUT/bench.err
  done
done
done
echo done > $OUT/DONE
