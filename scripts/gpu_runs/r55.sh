set -u
OUT=gpurun_out/r55; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for m in 0 1; do
  timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu-baseline --method $m > $OUT/bench_c1_m$m.json 2> $OUT/bench_c1_m$m.err
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches_c1_m$m.csv \
     python bench.py --config c1 --steps 4 --warmup 3 --no-cpu-baseline --method $m > $OUT/ncu_c1_m$m.log 2>&1
done
