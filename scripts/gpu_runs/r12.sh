set -u
bash scripts/gpu_round.sh r12 smoke ktests benchk ncuk
