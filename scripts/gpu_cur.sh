# int8 GDA fit: the shift prologue's loads in one round trip vs HEAD
OUT=gpurun_out/r371; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -m pytest tests -m gpu -q -x -k "gda or c3" --timeout 100 > $OUT/pytest_gda.log 2>&1; echo "rc=$?" >> $OUT/pytest_gda.log
for i in 1 2 3; do
  timeout 120 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/c3_new_$i.json 2>&1
  DLX_LIB_PATH=$PWD/build_old/libdlx.so timeout 120 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/c3_old_$i.json 2>&1
done
echo done > $OUT/DONE
