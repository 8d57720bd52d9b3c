# GDA combine with 256-thread blocks vs 1024 (HEAD): GDA tests + C3 A/B + launch list
OUT=gpurun_out/r368; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -m pytest tests -m gpu -q -x -k "gda or c3" --timeout 100 > $OUT/pytest_gda.log 2>&1; echo "rc=$?" >> $OUT/pytest_gda.log
for i in 1 2 3; do
  timeout 120 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/c3_new_$i.json 2>&1
  DLX_LIB_PATH=$PWD/build_old/libdlx.so timeout 120 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/c3_old_$i.json 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv --log-file $OUT/launches_c3.csv python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_l3.log 2>&1
echo done > $OUT/DONE
