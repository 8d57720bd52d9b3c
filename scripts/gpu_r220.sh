OUT=gpurun_out/r220; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_peer.py -m gpu -q -rf --timeout 800 --durations=10 > $OUT/pytest_peer.log 2>&1; echo "rc=$?" >> $OUT/pytest_peer.log
timeout 900 python scripts/program_times.py > $OUT/program_times.jsonl 2> $OUT/program_times.err
