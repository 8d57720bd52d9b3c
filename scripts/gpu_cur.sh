# GDA combine: the finalize reads the class sums from shared memory; tests, C3 bench, launch list
OUT=gpurun_out/r325; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py tests/test_gpu_program.py tests/test_gpu_sharded.py -m gpu -q -rf -x --timeout 300 -k "gda or c3" > $OUT/pytest_gda.log 2>&1; echo "rc=$?" >> $OUT/pytest_gda.log
for i in 1 2; do
  timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c3_$i.json 2>> $OUT/bench.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file $OUT/launches_c3.csv \
  python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_launch_c3.log 2>&1
echo done > $OUT/DONE
