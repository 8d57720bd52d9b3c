#!/bin/bash
# ncu full capture of the single-pass GDA fit kernel (gda_pass2_dmma_kernel<1>)
OUT=gpurun_out/r93; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gda_pass2 -s 4 -c 1 -o $OUT/prof_c3 \
  python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_c3.log 2>&1
