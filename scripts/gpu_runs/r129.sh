#!/bin/bash
# GDA operand tiles with interleaved (k, k+4) pair-rows: 16-byte fragment loads (4 per 6 DMMAs)
OUT=gpurun_out/r129; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_staged_programs.py tests/test_gpu_peer.py -m gpu -q -rf -k "gda or overlap or staged" > $OUT/pytest_gda.log 2>&1; echo "rc=$?" >> $OUT/pytest_gda.log
for i in 1 2 3; do timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_c3_$i.json 2> $OUT/bench_c3_$i.err; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gda_pass2" -s 4 -c 1 -o $OUT/prof_c3 python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline > $OUT/ncu_c3.log 2>&1
