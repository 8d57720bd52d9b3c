OUT=gpurun_out/r206; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
DLX_PROGRAM_PROFILE=1 timeout 300 python scripts/diag/c4_program_timing.py 10 > $OUT/timing.txt 2>&1
