# session 3 of round 2: re-confirm the restored tree on a fresh box
bash scripts/gpu_round.sh r300 smoke tests
OUT=gpurun_out/r300
for c in c4 c4shard8 c3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
