set -u
OUT=gpurun_out/r36; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -rf > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches_c3.csv \
   python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gda_pass2 -s 3 -c 1 -o $OUT/prof_gda2 \
   python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_gda2.log 2>&1
