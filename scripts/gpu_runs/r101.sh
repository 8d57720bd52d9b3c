#!/bin/bash
# flakiness sweep: the whole GPU suite three times, then the new kernels' tests ten times
OUT=gpurun_out/r101; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for i in 1 2 3; do
  timeout 900 python -m pytest tests -m gpu -q -x > $OUT/full_$i.log 2>&1; echo "rc=$?" >> $OUT/full_$i.log
done
for i in $(seq 1 10); do
  timeout 600 python -m pytest tests/test_gpu_peer.py tests/test_gpu_parity.py -q -x -k "peer or gda or groupby or shapes or c1 or screened" > $OUT/sub_$i.log 2>&1; echo "rc=$?" >> $OUT/sub_$i.log
done
