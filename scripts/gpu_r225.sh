OUT=gpurun_out/r225; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python scripts/diag/e2e_dropin_profile.py 2097152 64 64 > $OUT/e2e_shard8.json 2> $OUT/e2e_shard8_profile.txt
timeout 300 python scripts/diag/e2e_dropin_profile.py 65536 16 8 > $OUT/e2e_c1.json 2> $OUT/e2e_c1_profile.txt
for i in 1 2; do timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_c3_$i.json 2>> $OUT/bench.err; done
