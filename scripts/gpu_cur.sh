# A/B: small-kernel staging (one round of 16 loads vs the previous loop), C1 bench alternating
OUT=gpurun_out/r338; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for i in 1 2 3; do
  timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c1_new_$i.json 2>&1
  DLX_LIB_PATH=$PWD/build_old/libdlx.so timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/c1_old_$i.json 2>&1
done
echo done > $OUT/DONE
