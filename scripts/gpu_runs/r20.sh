set -u
OUT=gpurun_out/r20; mkdir -p $OUT
DLX_KMEANS_TRACE=1 DLX_KMEANS_PF=0 timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_pf0.json 2> $OUT/trace_pf0.err
