# final validation of the committed tree: smoke, full GPU suite, default bench, reference arm, C3
OUT=gpurun_out/r367; mkdir -p $OUT
bash scripts/gpu_round.sh r367 smoke tests benchref
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 > $OUT/bench_c3.json 2> $OUT/bench_c3.err
echo done > $OUT/DONE2
