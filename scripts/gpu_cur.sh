# per-class sums (inf-safe) in both fits: full GPU suite, smoke, C3 bench, launch list
OUT=gpurun_out/r353; mkdir -p $OUT
bash scripts/gpu_round.sh r353 smoke tests
for i in 1 2; do
  timeout 120 python bench.py --config c3 --steps 20 --warmup 3 > $OUT/c3_$i.json 2>&1
  DLX_GDA_I8=0 timeout 120 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/c3_dmma_$i.json 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file $OUT/launches_c3.csv python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_l.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:gda_fit_i8 -s 3 -c 1 -o $OUT/prof_c3_i8 python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_f.log 2>&1
echo done > $OUT/DONE2
