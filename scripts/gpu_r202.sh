OUT=gpurun_out/r203; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_program.py tests/test_staged_programs.py -m gpu -q -rf > $OUT/pytest_prog.log 2>&1; echo "rc=$?" >> $OUT/pytest_prog.log
timeout 600 python scripts/c4_staged.py 10 > $OUT/c4_staged.json 2> $OUT/c4_staged.err
