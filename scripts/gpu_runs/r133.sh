#!/bin/bash
# GDA fused class sums: predicated single add per element (branch) vs select-and-add (two adds)
OUT=gpurun_out/r133; mkdir -p $OUT
for V in branch sel branch sel; do
  cp scripts/gpu_runs/gda_$V.cu paper_1109_0778_b200/csrc/gda_dmma.cu
  make -s -j16 -C paper_1109_0778_b200 > $OUT/build.log 2>&1
  timeout 300 python bench.py --config c3 --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('$V', round(r['value'],1), round(r['roofline']['frac'],4))" >> $OUT/res.txt
done
cp scripts/gpu_runs/gda_branch.cu paper_1109_0778_b200/csrc/gda_dmma.cu
make -s -j16 -C paper_1109_0778_b200 > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -k gda > $OUT/pytest_gda.log 2>&1; echo "rc=$?" >> $OUT/pytest_gda.log
