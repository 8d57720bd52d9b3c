OUT=gpurun_out/r223; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_sharded.py -m gpu -q -rf --timeout 600 --durations=10 > $OUT/pytest_sharded.log 2>&1; echo "rc=$?" >> $OUT/pytest_sharded.log
