# r311: fp32-storage logreg: exact integer float->double, fp64-kernel block order; C3 program profile
OUT=gpurun_out/r311; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -k "logreg" > $OUT/pytest_logreg.log 2>&1; echo "rc=$?" >> $OUT/pytest_logreg.log
for c in l16f32 l16; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
DLX_PROGRAM_PROFILE=1 timeout 300 python scripts/diag/program_profile.py c3 > $OUT/c3_profile.txt 2>&1
echo done > $OUT/DONE
