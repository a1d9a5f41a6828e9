#!/bin/bash
# Timing ablations of the tensor-core pass (results are wrong by design): block period of the middle CTA with
# parts of the loop removed.  usage (under gpurun): bash tools/ablate.sh   (after tools/build_ablate.py)
for v in 0 1 2 4 8 16 6 31; do
  echo -n "ablate=$v: "
  FOE_LIB=paper_1609_05722_b200/libfoe_b200_ab$v.so python tools/diag_times.py 2>&1 | python -c "
import sys,re
txt=sys.stdin.read()
rows=re.findall(r'\[\s*(-?\d+)\s+(-?\d+)\s+(-?\d+)\s+(-?\d+)\s+(-?\d+)\s+(-?\d+)\s+(-?\d+)\s+(-?\d+)\s+(-?\d+)\s+(-?\d+)\]', txt)
f=[int(r[0]) for r in rows[:18]]
print('fwd issued block 4 -> 16:', f[4], f[16], 'period', (f[16]-f[4])/12)
"
done
