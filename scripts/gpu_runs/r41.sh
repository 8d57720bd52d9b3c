set -u
OUT=gpurun_out/r41; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python bench.py --config c4shard8 --steps 50 --warmup 5 --no-cpu-baseline > $OUT/bench_shard8.json 2> $OUT/bench_shard8.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches_shard8.csv \
   python bench.py --config c4shard8 --steps 4 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
