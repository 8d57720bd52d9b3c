set -u
OUT=gpurun_out/r25; mkdir -p $OUT
bash scripts/gpu_round.sh r25 ktests benchk
make -s -B -j8 -C paper_1109_0778_b200 NVFLAGS="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -DDLX_KMEANS_TRACE" > $OUT/trace_build.log 2>&1
DLX_KMEANS_TRACE=1 timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_trace.json 2> $OUT/trace.err
