set -u
OUT=gpurun_out/r21; mkdir -p $OUT
for pf in 0 1 3; do
  DLX_KMEANS_PF=$pf timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_pf$pf.json 2> $OUT/bench_pf$pf.err
done
