set -u
bash scripts/gpu_round.sh r31 smoke tests benchk ncuk
