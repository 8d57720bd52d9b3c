#!/bin/bash
# ncu full capture of the screened kernel after the L2 prefetch change
OUT=gpurun_out/r119; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:kmeans_screened -s 3 -c 1 -o $OUT/prof_kmeans \
  python bench.py --config c4 --steps 4 --warmup 3 --no-cpu-baseline > $OUT/ncu.log 2>&1
