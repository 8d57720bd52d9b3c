#!/bin/bash
# compute-sanitizer memcheck on the executor's overlapped loops (stream-ordered frees, pinned staging)
# and on the GDA fit with the pair-row operand layout
OUT=gpurun_out/r135; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_staged_programs.py -m gpu -q -x -k "not kmeans_n65536 and not kmeans_n4096" > $OUT/memcheck_staged.txt 2>&1; echo "rc=$?" >> $OUT/memcheck_staged.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "gda_shapes or gda_fit_matches" > $OUT/memcheck_gda.txt 2>&1; echo "rc=$?" >> $OUT/memcheck_gda.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "gda_shapes and 37893" > $OUT/racecheck_gda.txt 2>&1; echo "rc=$?" >> $OUT/racecheck_gda.txt
