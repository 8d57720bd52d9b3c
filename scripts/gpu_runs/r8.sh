set -u
OUT=gpurun_out/r8; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
DLX_KMEANS_TRACE=1 timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_trace.json 2> $OUT/trace.err
timeout 600 python -m pytest tests -m gpu -q -rf -k "staged" > $OUT/pytest_staged.log 2>&1
timeout 300 oracle/_ref/run_staged > $OUT/run_staged.log 2>&1; echo "rc=$?" >> $OUT/run_staged.log
