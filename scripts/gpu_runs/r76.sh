#!/bin/bash
# GDA pass 2: shared-index block triples for d = 64 (4 fragment loads per 3 DMMA)
OUT=gpurun_out/r76; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -rf -k "gda" > $OUT/pytest_gda.log 2>&1; echo "rc=$?" >> $OUT/pytest_gda.log
timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gda_pass2 -c 3 --csv --log-file $OUT/launches.csv \
  python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu2.log 2>&1
