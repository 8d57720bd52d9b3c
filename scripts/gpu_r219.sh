OUT=gpurun_out/r219; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 600 -x --durations=10 > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for i in 1 2; do
timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_c3_k64_$i.json 2> $OUT/bench_c3.err
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gda_fit64 -c 1 -o $OUT/prof_c3 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu.log 2>&1
