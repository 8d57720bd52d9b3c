# early L2 prefetch of the first tiles before the PDL wait: A/B vs the committed kernel; N=2 code path on one GPU
OUT=gpurun_out/r320; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -x --timeout 300 -k "kmeans or screened or c4" > $OUT/pytest_kmeans.log 2>&1; echo "rc=$?" >> $OUT/pytest_kmeans.log
for i in 1 2 3; do
for v in acc3 new; do
  if [ $v = new ]; then L=""; else L=paper_1109_0778_b200/build_$v/libdlx.so; fi
  for c in c4 c4shard8; do
    DLX_LIB_PATH=$L timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_${c}_${v}_$i.json 2>> $OUT/bench.err
  done
done
done
DLX_BENCH_SHARED_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 5 --warmup 3 > $OUT/bench_n2_shared.json 2> $OUT/bench_n2_shared.err; echo "rc=$?" >> $OUT/bench_n2_shared.err
echo done > $OUT/DONE
