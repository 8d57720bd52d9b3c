#!/bin/bash
# bench.py N=2 code path on one device (DLX_BENCH_SHARED_DEVICE: gloo plumbing + peer exchange)
OUT=gpurun_out/r107; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for c in c1 c4shard8 c2 c3 c5; do
  DLX_BENCH_SHARED_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 3 --warmup 3 --config $c --comm peer \
    > $OUT/n2_$c.json 2> $OUT/n2_$c.err
  echo "$c rc=$?" >> $OUT/rc.txt
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 3 --config c1 > $OUT/n2_ref.json 2> $OUT/n2_ref.err
echo "ref rc=$?" >> $OUT/rc.txt
