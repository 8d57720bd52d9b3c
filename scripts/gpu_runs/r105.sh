#!/bin/bash
# sharded GDA: per-rank single-pass fits pooled through the exchange (world 2 on one device); c3 bench
OUT=gpurun_out/r105; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_peer.py tests/test_gpu_parity.py -q -rf -k "peer or gda" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c3.json 2>$OUT/err
