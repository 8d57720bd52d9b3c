set -u
OUT=gpurun_out/r19; mkdir -p $OUT
for pf in 0 2 3 5 8; do
  DLX_KMEANS_TRACE=1 DLX_KMEANS_PF=$pf timeout 300 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_pf$pf.json 2> $OUT/trace_pf$pf.err
done
