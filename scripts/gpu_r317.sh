# r317: deferred prints formatted on a host pool; staged-program tests and drop-in program times
OUT=gpurun_out/r317; mkdir -p $OUT
timeout 900 python -m pytest tests/test_staged_programs.py tests/test_gpu_program.py tests/test_gpu_sharded.py -m gpu -q -rf > $OUT/pytest_prog.log 2>&1; echo "rc=$?" >> $OUT/pytest_prog.log
timeout 300 python scripts/program_times.py c1 c2 c3 c4 > $OUT/program_times.jsonl 2> $OUT/program_times.err
DLX_PROGRAM_PROFILE=1 timeout 300 python scripts/diag/program_profile.py c3 > $OUT/c3_profile.txt 2>&1
echo done > $OUT/DONE
