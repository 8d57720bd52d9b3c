# A/B: GDA class sums on aux warps (DLX_G64_AUX_SUMS=1, build_aux/) vs default
OUT=gpurun_out/r335; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
DLX_LIB_PATH=$PWD/build_aux/libdlx.so timeout 400 python -m pytest tests -m gpu -q -x -k "gda" --timeout 120 > $OUT/pytest_gda_aux.log 2>&1; echo "rc=$?" >> $OUT/pytest_gda_aux.log
for i in 1 2; do
  timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/c3_def_$i.json 2>&1
  DLX_LIB_PATH=$PWD/build_aux/libdlx.so timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/c3_aux_$i.json 2>&1
done
grep -q "rc=0" $OUT/pytest_gda_aux.log && DLX_LIB_PATH=$PWD/build_aux/libdlx.so timeout 400 ncu --set full --clock-control none --import-source on -k regex:gda_fit64 -s 4 -c 1 -o $OUT/prof_c3_aux python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu.log 2>&1
echo done > $OUT/DONE
