set -u
mkdir -p gpurun_out/r18
./scripts/mb/f2i > gpurun_out/r18/f2i.txt 2>&1
bash scripts/gpu_round.sh r18 smoke ktests benchk ncuk
