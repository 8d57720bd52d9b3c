set -u
bash scripts/gpu_round.sh r17 smoke ktests benchk ncuk
