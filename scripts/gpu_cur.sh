# compute-sanitizer synccheck / racecheck / memcheck after the split-barrier fixes
OUT=gpurun_out/r364; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 compute-sanitizer --tool synccheck --kernel-name kns=gda_fit --print-limit 10 python scripts/diag/san_gda_i8.py > $OUT/san_gda_synccheck.txt 2>&1; echo "rc=$?" >> $OUT/san_gda_synccheck.txt
DLX_GDA_I8=0 timeout 600 compute-sanitizer --tool synccheck --kernel-name kns=gda_fit --print-limit 10 python scripts/diag/san_gda_i8.py > $OUT/san_gda_dmma_synccheck.txt 2>&1; echo "rc=$?" >> $OUT/san_gda_dmma_synccheck.txt
for t in synccheck memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $t --kernel-name kns=kmeans_screened --print-limit 10 python scripts/diag/san_kmeans.py > $OUT/san_kmeans_$t.txt 2>&1; echo "rc=$?" >> $OUT/san_kmeans_$t.txt
done
timeout 300 python -m pytest tests -m gpu -q -x -k "gda or screened or c4 or c3" --timeout 200 > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 200 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/c4.json 2>&1
echo done > $OUT/DONE
