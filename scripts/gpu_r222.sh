OUT=gpurun_out/r222; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_sharded.py -m gpu -q -rf --timeout 600 -x --durations=10 > $OUT/pytest_sharded.log 2>&1; echo "rc=$?" >> $OUT/pytest_sharded.log
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 600 --durations=10 --ignore=tests/test_gpu_sharded.py > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python scripts/program_times.py c1 c2 c3 > $OUT/program_times.jsonl 2> $OUT/program_times.err
