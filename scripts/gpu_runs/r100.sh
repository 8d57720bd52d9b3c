#!/bin/bash
# small k-means kernel: 8 loads in flight in the tile staging
OUT=gpurun_out/r100; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "kmeans or c1" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python bench.py --config c1 --steps 200 --warmup 10 --no-cpu-baseline > $OUT/bench_c1.json 2>$OUT/err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches_c1.csv \
  python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/ncu.log 2>&1
timeout 600 python scripts/kmeans_crossover.py > $OUT/crossover.txt 2>&1
