set -u
bash scripts/gpu_round.sh r51 smoke tests bench benchref ncu
timeout 300 python bench.py --config c4shard8 --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/r51/bench_c4shard8.json 2> gpurun_out/r51/bench_c4shard8.err
