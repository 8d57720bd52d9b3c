# C1 warm-cache profile of the small kernel + combine (ncu --cache-control none)
OUT=gpurun_out/r340; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -c 20 --csv --log-file $OUT/launches_c1_warm.csv python bench.py --config c1 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_l.log 2>&1
timeout 300 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"kmeans_small|combine_kmeans" -s 6 -c 2 -o $OUT/prof_c1_warm python bench.py --config c1 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_f.log 2>&1
echo done > $OUT/DONE
