#!/bin/bash
# single-pass GDA fit (shifted DMMA scatter + rank-1 correction, device-side certified fallback)
OUT=gpurun_out/r80; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "gda" > $OUT/pytest_gda.log 2>&1; echo "rc=$?" >> $OUT/pytest_gda.log
timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches.csv \
  python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu2.log 2>&1
