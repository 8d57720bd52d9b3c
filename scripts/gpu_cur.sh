# validation of the committed state: smoke, full GPU suite, default bench (C4), C3/C1 lines, launch lists
OUT=gpurun_out/r360; mkdir -p $OUT
bash scripts/gpu_round.sh r360 smoke tests
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for c in c3 c1 c2 l16 c5 c4shard8; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file $OUT/launches_c3.csv python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_l3.log 2>&1
echo done > $OUT/DONE2
