set -u
bash scripts/gpu_round.sh r22 ktests benchk
