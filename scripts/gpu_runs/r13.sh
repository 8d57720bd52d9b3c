set -u
bash scripts/gpu_round.sh r13 smoke ktests benchk ncuk
