# drop-in e2e regression hunt: host print pool on / off, raw-pointer lazies; C4 e2e and program times
OUT=gpurun_out/r327; mkdir -p $OUT
for i in 1 2; do
  timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c4_pool_$i.json 2> $OUT/bench_c4_pool_$i.err
  DLX_HOST_POOL=0 timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c4_nopool_$i.json 2> $OUT/bench_c4_nopool_$i.err
done
timeout 300 python scripts/program_times.py c3 c4 > $OUT/program_times_pool.jsonl 2> $OUT/program_times.err
DLX_HOST_POOL=0 timeout 300 python scripts/program_times.py c3 c4 > $OUT/program_times_nopool.jsonl 2>> $OUT/program_times.err
timeout 300 python scripts/diag/e2e_dropin_profile.py 16777216 64 64 > $OUT/e2e_c4.json 2> $OUT/e2e_c4_profile.txt
echo done > $OUT/DONE
