#!/bin/bash
# C4 through the drop-in executor (directly built staged descriptor), GPU tests, executor timings
OUT=gpurun_out/r130; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python scripts/c4_staged.py > $OUT/c4_staged.json 2> $OUT/c4_staged.err; echo "rc=$?" >> $OUT/c4_staged.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
