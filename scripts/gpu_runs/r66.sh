#!/bin/bash
OUT=gpurun_out/r66; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 400 python -m pytest tests/test_gpu_peer.py -q -rf > $OUT/pytest_peer.log 2>&1; echo "rc=$?" >> $OUT/pytest_peer.log
