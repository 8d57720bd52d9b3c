#!/bin/bash
# GroupBy K=65536 cluster path: remote DSMEM atomics vs lockstep double-read with local atomics
OUT=gpurun_out/r86; mkdir -p $OUT
BASE="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
for R in 0 1; do
  make -C paper_1109_0778_b200 -j16 NVFLAGS="$BASE -DDLX_GB_PAIR_REMOTE=$R" > $OUT/build_$R.log 2>&1
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -rf -k "groupby" > $OUT/pytest_$R.log 2>&1; echo "rc=$?" >> $OUT/pytest_$R.log
  timeout 300 python bench.py --config c5k65536 --steps 10 --warmup 3 --no-cpu-baseline 2>$OUT/err_$R | python -c "import json,sys; r=json.loads(sys.stdin.readline()); print('remote=$R', round(r['value'],1), r['ms_per_step'], round(r['roofline']['frac'],4))" >> $OUT/res.txt
done
make -C paper_1109_0778_b200 -j16 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:groupby -c 4 --csv --log-file $OUT/ncu.csv \
  python bench.py --config c5k65536 --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu.log 2>&1
