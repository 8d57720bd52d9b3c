#!/bin/bash
# executor: host mirrors of small vectors (batched element reads / updates) — parity + A/B timing
OUT=gpurun_out/r110; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_staged_programs.py -q -rf -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python scripts/time_programs.py > $OUT/times.txt 2>&1
