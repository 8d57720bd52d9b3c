# k-means L2 prefetch distance re-tune after the three-accumulator screen (0 / 2 / 3 / 4 tiles); the
# two-thread print-formatting test
OUT=gpurun_out/r329; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_program.py -m gpu -q -rf --timeout 300 -k "parallel_print" > $OUT/pytest_pool.log 2>&1; echo "rc=$?" >> $OUT/pytest_pool.log
for i in 1 2; do
for v in cur l2a2 l2a4 l2a0; do
  if [ $v = cur ]; then L=""; else L=paper_1109_0778_b200/build_$v/libdlx.so; fi
  for c in c4 c4shard8; do
    DLX_LIB_PATH=$L timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_${c}_${v}_$i.json 2>> $OUT/bench.err
  done
done
done
echo done > $OUT/DONE
