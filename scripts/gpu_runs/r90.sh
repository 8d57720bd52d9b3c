#!/bin/bash
# small-problem direct k-means kernel (exact chain, counting-sort segmented fold)
OUT=gpurun_out/r90; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -x -k "kmeans or c1 or c4" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python bench.py --config c1 --steps 200 --warmup 10 --no-cpu-baseline > $OUT/bench_c1.json 2>$OUT/err
timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c4.json 2>>$OUT/err
timeout 900 python scripts/kmeans_crossover.py > $OUT/crossover.txt 2>&1
