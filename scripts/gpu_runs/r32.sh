set -u
bash scripts/gpu_round.sh r32 bench benchref ncu
