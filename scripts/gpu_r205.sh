OUT=gpurun_out/r205; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python scripts/diag/c4_program_timing.py 10 > $OUT/timing.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches.csv python scripts/diag/c4_program_timing.py 2 > $OUT/ncu.log 2>&1
