set -u
bash scripts/gpu_round.sh r16 smoke ktests benchk ncuk
