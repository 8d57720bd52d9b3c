# final full validation: every GPU test, smoke, default bench line
bash scripts/gpu_round.sh r332 smoke tests
OUT=gpurun_out/r332
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
