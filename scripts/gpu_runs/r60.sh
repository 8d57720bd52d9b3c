set -u
bash scripts/gpu_round.sh r60 smoke tests bench benchref ncu
timeout 300 python bench.py --config c4shard8 --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/r60/bench_c4shard8.json 2> gpurun_out/r60/bench_c4shard8.err
timeout 300 python bench.py --config c4 --steps 50 --warmup 5 > gpurun_out/r60/bench_c4_long.json 2> gpurun_out/r60/bench_c4_long.err
