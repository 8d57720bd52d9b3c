#!/bin/bash
OUT=gpurun_out/r64; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 200 python -m pytest tests/test_gpu_peer.py -q -rf -x -s -k world1 > $OUT/pytest_world1.log 2>&1; echo "rc=$?" >> $OUT/pytest_world1.log
timeout 150 python scripts/diag/peer_diag.py > $OUT/diag.log 2>&1; echo "rc=$?" >> $OUT/diag.log
nvidia-smi -q | grep -i -A3 "compute mode\|MPS" > $OUT/smi.txt 2>&1
