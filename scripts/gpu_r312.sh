# r312: round profiles — ncu launch list (C4) and --set full captures of the dominant kernels
# (k-means screened C4, GDA fit C3, logreg L16 fp64 and fp32 storage, GroupBy C5); fp32 row-group A/B
OUT=gpurun_out/r312; mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
for v in f32g3 f32g4; do
  DLX_LIB_PATH=paper_1109_0778_b200/build_$v/libdlx.so timeout 300 python bench.py --config l16f32 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_l16f32_$v.json 2>> $OUT/bench.err
done
timeout 300 python bench.py --config l16f32 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_l16f32_g2.json 2>> $OUT/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $OUT/launches_c4.csv \
  python bench.py --config c4 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_launch_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kmeans_screened -s 3 -c 1 -o $OUT/prof_c4 \
  python bench.py --config c4 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_full_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gda_fit64 -s 3 -c 1 -o $OUT/prof_c3 \
  python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_full_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:logreg_grad -s 4 -c 1 -o $OUT/prof_l16 \
  python bench.py --config l16 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_full_l16.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:logreg_grad -s 4 -c 1 -o $OUT/prof_l16f32 \
  python bench.py --config l16f32 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_full_l16f32.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:groupby_smem -s 4 -c 1 -o $OUT/prof_c5 \
  python bench.py --config c5 --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_full_c5.log 2>&1
echo done > $OUT/DONE
