#!/bin/bash
# GDA pass 2 v2 (bulk-TMA ring, 12 warps x 3 blocks): parity + c3 bench + ncu
OUT=gpurun_out/r69; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -rf -k "gda" > $OUT/pytest_gda.log 2>&1; echo "rc=$?" >> $OUT/pytest_gda.log
timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gda_pass2 -s 2 -c 1 -o $OUT/prof_gda \
  python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu.log 2>&1
