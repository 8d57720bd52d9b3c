# r318: host pool made immortal (exit hung in r317: a condition variable destroyed with waiters);
# lazy chunks; staged / program / sharded tests, drop-in program times, C3 profile, reference arm
OUT=gpurun_out/r318; mkdir -p $OUT
timeout 900 python -m pytest tests/test_staged_programs.py tests/test_gpu_program.py tests/test_gpu_sharded.py -m gpu -q -rf --timeout 300 > $OUT/pytest_prog.log 2>&1; echo "rc=$?" >> $OUT/pytest_prog.log
timeout 300 python scripts/program_times.py c1 c2 c3 c4 > $OUT/program_times.jsonl 2> $OUT/program_times.err; echo "rc=$?" >> $OUT/program_times.err
DLX_PROGRAM_PROFILE=1 timeout 300 python scripts/diag/program_profile.py c3 > $OUT/c3_profile.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref_c4.json 2> $OUT/bench_ref_c4.err
echo done > $OUT/DONE
