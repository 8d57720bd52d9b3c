# r316: full GPU suite + smoke on the current tree; default bench lines
bash scripts/gpu_round.sh r316 smoke tests
OUT=gpurun_out/r316
for c in c4 c4shard8 c3 l16 l16f32 c2 c1 c5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 300 python scripts/program_times.py c1 c2 c3 c4 > $OUT/program_times.jsonl 2> $OUT/program_times.err
