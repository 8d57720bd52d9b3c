OUT=gpurun_out/r214; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 600 --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
oracle/_ref/run_staged > $OUT/run_staged.txt 2>&1; echo "rc=$?" >> $OUT/run_staged.txt
timeout 300 python scripts/c4_staged.py > $OUT/c4_staged.json 2> $OUT/c4_staged.err
timeout 300 python scripts/time_programs.py > $OUT/time_programs.txt 2>&1
