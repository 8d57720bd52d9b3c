set -u
OUT=gpurun_out/r33; mkdir -p $OUT
bash scripts/gpu_round.sh r33 smoke tests benchk
F="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr"
make -s -B -j8 -C paper_1109_0778_b200 NVFLAGS="$F -DDLX_KMEANS_EPI_X8" > $OUT/build_x8.log 2>&1
timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_x8.json 2> $OUT/bench_x8.err
