#!/bin/bash
# peer-memory fused allreduce: world-2 on one device + world-1 epilogues; then the c4 bench line
OUT=gpurun_out/r63; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_peer.py -q -rf -x > $OUT/pytest_peer.log 2>&1; echo "rc=$?" >> $OUT/pytest_peer.log
timeout 300 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err
