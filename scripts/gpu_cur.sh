# C3 / C1 drop-in host timelines after the host-cost trims
OUT=gpurun_out/r333; mkdir -p $OUT
DLX_PROGRAM_PROFILE=1 timeout 300 python scripts/diag/program_profile.py c3 > $OUT/c3_profile.txt 2>&1
DLX_PROGRAM_PROFILE=1 timeout 300 python scripts/diag/program_profile.py c1 > $OUT/c1_profile.txt 2>&1
echo done > $OUT/DONE
