#!/bin/bash
# trap precedence of overlapped loops; staged tests
OUT=gpurun_out/r136; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_staged_programs.py -m gpu -q -rf > $OUT/pytest_staged.log 2>&1; echo "rc=$?" >> $OUT/pytest_staged.log
