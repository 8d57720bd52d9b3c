# final validation after the stage change: smoke, full GPU suite, default bench, C3, reference arm
OUT=gpurun_out/r370; mkdir -p $OUT
bash scripts/gpu_round.sh r370 smoke tests benchref
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 > $OUT/bench_c3.json 2> $OUT/bench_c3.err
echo done > $OUT/DONE2
