OUT=gpurun_out/r221; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
bash scripts/build_variant.sh r128 "-DDLX_G64_ROWS=128" > $OUT/build_r128.log 2>&1
timeout 900 python -m pytest tests/test_gpu_peer.py -m gpu -q -rf --timeout 800 --durations=10 > $OUT/pytest_peer.log 2>&1; echo "rc=$?" >> $OUT/pytest_peer.log
for i in 1 2; do
timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_c3_r64_$i.json 2>> $OUT/bench.err
DLX_LIB_PATH=paper_1109_0778_b200/build_r128/libdlx.so timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_c3_r128_$i.json 2>> $OUT/bench.err
done
DLX_LIB_PATH=paper_1109_0778_b200/build_r128/libdlx.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k gda > $OUT/pytest_gda_r128.log 2>&1
for c in c2 c3; do DLX_PROGRAM_PROFILE=1 timeout 300 python scripts/diag/program_profile.py $c > /dev/null 2> $OUT/profile_$c.txt; done
