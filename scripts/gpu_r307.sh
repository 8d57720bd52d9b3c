# r307: per-tile traces, committed 3-accumulator kernel vs the two-stage TMEM hand-off
OUT=gpurun_out/r307; mkdir -p $OUT
for v in trace3 trace2; do
  for n in 16777216 2097152; do
    DLX_LIB_PATH=paper_1109_0778_b200/build_$v/libdlx.so DLX_KMEANS_TRACE=1 timeout 300 python scripts/diag/kmeans_trace.py $n > $OUT/trace_${v}_$n.txt 2>&1
  done
done
echo done > $OUT/DONE
