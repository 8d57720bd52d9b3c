# r310: fp32-storage logreg with 16 packed rows in flight per warp (d <= 64)
OUT=gpurun_out/r310; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -k "logreg" > $OUT/pytest_logreg.log 2>&1; echo "rc=$?" >> $OUT/pytest_logreg.log
for c in l16f32 l16 c2; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
echo done > $OUT/DONE
