#!/bin/bash
# One gpurun session: build, smoke, GPU parity tests, bench lines, ncu launch list + full capture.
# Usage (from repo root, under gpurun): bash scripts/gpu_round.sh [tag] [what...]
set -u
TAG=${1:-r1}
shift || true
WHAT=${*:-"smoke tests bench ncu"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> $OUT/nproc.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || echo "BUILD FAILED" >> $OUT/build.log
for w in $WHAT; do
  case $w in
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log ;;
    ktests) timeout 600 python -m pytest tests -m gpu -q -rf -x -k "screened or c1_step or c4 or kmeans or staged" > $OUT/pytest_kmeans.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_kmeans.log ;;
    benchk) timeout 600 python bench.py --config c4 --steps 20 --warmup 3 > $OUT/bench_c4.json 2> $OUT/bench_c4.err
            timeout 600 python bench.py --config c1 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c1.json 2> $OUT/bench_c1.err ;;
    ncuk) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $OUT/launches_c4.csv \
           python bench.py --config c4 --steps 4 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_bench.log 2>&1
         timeout 1200 ncu --set full --clock-control none --import-source on -k regex:kmeans_screened -s 3 -c 1 -o $OUT/prof_kmeans \
           python bench.py --config c4 --steps 4 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_kmeans.log 2>&1 ;;
    tests) timeout 1800 python -m pytest tests -m gpu -q -rf --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log ;;
    bench) for c in c4 c1 c2 l16 c3 c5 c5k65536 c4shard8; do
             timeout 600 python bench.py --config $c --steps 10 --warmup 3 > $OUT/bench_$c.json 2> $OUT/bench_$c.err
           done ;;
    benchref) timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref_c4.json 2> $OUT/bench_ref_c4.err ;;
    ncu) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $OUT/launches_c4.csv \
           python bench.py --config c4 --steps 4 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_bench.log 2>&1
         timeout 1200 ncu --set full --clock-control none --import-source on -k regex:kmeans_screened -s 3 -c 1 -o $OUT/prof_kmeans \
           python bench.py --config c4 --steps 4 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_kmeans.log 2>&1
         for c in c5 l16 c3; do
           timeout 900 ncu --set full --clock-control none --import-source on -k regex:"groupby_smem|logreg_grad|gda_fit64" -s 4 -c 1 -o $OUT/prof_$c \
             python bench.py --config $c --steps 4 --warmup 3 --no-cpu-baseline > $OUT/ncu_full_$c.log 2>&1
         done ;;
  esac
done
echo done > $OUT/DONE
