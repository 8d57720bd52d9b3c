OUT=gpurun_out/r200; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python scripts/c4_staged.py > $OUT/c4_staged.json 2> $OUT/c4_staged.err
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err
nproc > $OUT/nproc.txt
