#!/bin/bash
# DEG overlap: staged-program tests, smoke, program timings (overlap / serial / per-element)
OUT=gpurun_out/r128; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_staged_programs.py tests/test_abi.py -m gpu -q -rf > $OUT/pytest_staged.log 2>&1; echo "rc=$?" >> $OUT/pytest_staged.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 900 python scripts/time_programs.py > $OUT/times.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
