#!/bin/bash
# executor: read-through pages for large vectors, pool keeps 32 GB mapped; C4 through the executor
OUT=gpurun_out/r132; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_staged_programs.py tests/test_abi.py -m gpu -q -rf > $OUT/pytest_staged.log 2>&1; echo "rc=$?" >> $OUT/pytest_staged.log
timeout 600 python scripts/c4_staged.py > $OUT/c4_staged.json 2> $OUT/c4_staged.err; echo "rc=$?" >> $OUT/c4_staged.err
timeout 900 python scripts/time_programs.py > $OUT/times.txt 2>&1
