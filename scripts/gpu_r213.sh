OUT=gpurun_out/r213; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_program.py tests/test_staged_programs.py -m gpu -q -rf --timeout 600 > $OUT/pytest_prog.log 2>&1; echo "rc=$?" >> $OUT/pytest_prog.log
oracle/_ref/run_staged > $OUT/run_staged.txt 2>&1; echo "rc=$?" >> $OUT/run_staged.txt
