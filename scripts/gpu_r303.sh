# r303: batched record loads in the flush; traces of base / acc4 / acc3 (new) at C4 and the 2M shard
OUT=gpurun_out/r303; mkdir -p $OUT
for v in basetrace trace4 trace; do
  for n in 16777216 2097152; do
    DLX_LIB_PATH=paper_1109_0778_b200/build_$v/libdlx.so DLX_KMEANS_TRACE=1 timeout 300 python scripts/diag/kmeans_trace.py $n > $OUT/trace_${v}_$n.txt 2>&1
  done
done
for i in 1 2; do
for v in base acc4 new; do
  if [ $v = new ]; then L=""; else L=paper_1109_0778_b200/build_$v/libdlx.so; fi
  for c in c4 c4shard8; do
    DLX_LIB_PATH=$L timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_${c}_${v}_$i.json 2>> $OUT/bench.err
  done
done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_program.py -m gpu -q -rf -x -k "kmeans or screened or c4 or c1" > $OUT/pytest_kmeans.log 2>&1; echo "rc=$?" >> $OUT/pytest_kmeans.log
echo done > $OUT/DONE
