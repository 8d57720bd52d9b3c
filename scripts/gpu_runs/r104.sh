#!/bin/bash
# racecheck with a high print limit: which shared-memory hand-offs does it flag?
OUT=gpurun_out/r104; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 200000 python scripts/diag/sanitize_screened.py > $OUT/racecheck.log 2>&1; echo "rc=$?" >> $OUT/racecheck.log
timeout 900 compute-sanitizer --tool memcheck python scripts/diag/sanitize_screened.py > $OUT/memcheck.log 2>&1; echo "rc=$?" >> $OUT/memcheck.log
python - > $OUT/pairs.txt <<'PY'
import re,collections
txt=open('gpurun_out/r104/racecheck.log').read()
pairs=collections.Counter()
for m in re.finditer(r'Potential (\w+) hazard.*?\n.*?(Write|Read) Thread.*?in (\S+):(\d+)\n.*?(Write|Read) Thread.*?in (\S+):(\d+)', txt):
    pairs[(m.group(1), m.group(2), m.group(3)+':'+m.group(4), m.group(5), m.group(6)+':'+m.group(7))]+=1
for k,v in pairs.most_common(): print(v, k)
PY
gzip -f $OUT/racecheck.log
