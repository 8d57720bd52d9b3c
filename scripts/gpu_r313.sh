# r313: conversion microbenchmark; k-means converters with integer floor_scaled vs fma_rd + F2I
OUT=gpurun_out/r313; mkdir -p $OUT
./scripts/mb/conv > $OUT/conv_mb.txt 2>&1
DLX_LIB_PATH=paper_1109_0778_b200/build_intconv/libdlx.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -x -k "kmeans or screened or c4 or c1" > $OUT/pytest_intconv.log 2>&1; echo "rc=$?" >> $OUT/pytest_intconv.log
for i in 1 2 3; do
for v in base intconv; do
  if [ $v = base ]; then L=""; else L=paper_1109_0778_b200/build_$v/libdlx.so; fi
  for c in c4 c4shard8; do
    DLX_LIB_PATH=$L timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_${c}_${v}_$i.json 2>> $OUT/bench.err
  done
done
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file $OUT/launches_c3.csv \
  python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_launch_c3.log 2>&1
echo done > $OUT/DONE
