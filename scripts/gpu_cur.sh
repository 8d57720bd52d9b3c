# d = 64 converters with 8 columns per lane (8-byte plane stores) vs the committed kernel; smoke
OUT=gpurun_out/r323; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_program.py -m gpu -q -rf -x --timeout 300 -k "kmeans or screened or c4 or c1" > $OUT/pytest_kmeans.log 2>&1; echo "rc=$?" >> $OUT/pytest_kmeans.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
for i in 1 2 3; do
for v in acc3 new; do
  if [ $v = new ]; then L=""; else L=paper_1109_0778_b200/build_$v/libdlx.so; fi
  for c in c4 c4shard8; do
    DLX_LIB_PATH=$L timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_${c}_${v}_$i.json 2>> $OUT/bench.err
  done
done
done
echo done > $OUT/DONE
