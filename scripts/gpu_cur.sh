# int8 GDA fit: pass-0 fetch before the plane-stage wait; GDA tests + C3 bench + profile
OUT=gpurun_out/r359; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python -m pytest tests -m gpu -q -x -k "gda or c3" --timeout 100 > $OUT/pytest_gda.log 2>&1; echo "rc=$?" >> $OUT/pytest_gda.log
for i in 1 2; do
  timeout 120 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/c3_$i.json 2>&1
done
timeout 400 ncu --set full --clock-control none --import-source on -k regex:gda_fit_i8 -s 3 -c 1 -o $OUT/prof_c3_i8 python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_f.log 2>&1
echo done > $OUT/DONE
