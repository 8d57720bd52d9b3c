OUT=gpurun_out/r212; mkdir -p $OUT
nproc > $OUT/nproc.txt; free -g >> $OUT/nproc.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 600 --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > $OUT/bench_ref_c4.json 2> $OUT/bench_ref_c4.err
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 > $OUT/bench_c3.json 2> $OUT/bench_c3.err
