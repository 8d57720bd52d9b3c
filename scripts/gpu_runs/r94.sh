#!/bin/bash
# GDA centring: all row loads issued before use
OUT=gpurun_out/r94; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -rf -k "gda" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python bench.py --config c3 --steps 30 --warmup 3 --no-cpu-baseline > $OUT/bench_c3.json 2>$OUT/err
