# headline-shape unfused program through the executor's fusion on the B200
OUT=gpurun_out/r330; mkdir -p $OUT
timeout 900 python -m pytest tests/test_staged_programs.py -m gpu -q -rf --timeout 600 -k "headline or unfused or executor_fusion" -s > $OUT/pytest_headline.log 2>&1; echo "rc=$?" >> $OUT/pytest_headline.log
echo done > $OUT/DONE
