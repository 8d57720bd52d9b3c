# r306: two-stage screen TMEM hand-off (HH released first) vs the committed 3-accumulator kernel
OUT=gpurun_out/r306; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -x -k "kmeans or screened or c4 or c1" > $OUT/pytest_kmeans.log 2>&1; echo "rc=$?" >> $OUT/pytest_kmeans.log
for i in 1 2 3; do
for v in acc3 new; do
  if [ $v = new ]; then L=""; else L=paper_1109_0778_b200/build_$v/libdlx.so; fi
  for c in c4 c4shard8; do
    DLX_LIB_PATH=$L timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_${c}_${v}_$i.json 2>> $OUT/bench.err
  done
done
done
echo done > $OUT/DONE
