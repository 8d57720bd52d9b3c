#!/bin/bash
# C4 through the drop-in executor: pool keep threshold 0.25 GB (default) vs 32 GB
OUT=gpurun_out/r131; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python scripts/c4_staged.py > $OUT/c4_staged.json 2> $OUT/c4_staged.err; echo "rc=$?" >> $OUT/c4_staged.err
DLX_POOL_KEEP_GB=32 timeout 600 python scripts/c4_staged.py > $OUT/c4_staged_keep32.json 2> $OUT/c4_staged_keep32.err; echo "rc=$?" >> $OUT/c4_staged_keep32.err
