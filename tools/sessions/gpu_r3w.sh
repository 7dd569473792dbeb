#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python tools/build_variants.py fr1=GML_FREE_RUN=1 fr0=GML_FREE_RUN=0 > $OUT/bv.log 2>&1; echo "build=$?"
for r in 1 2; do
 for V in fr1 fr0; do
  GML_LIB=build/libgml_$V.so GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 1 > $OUT/w_$V.log 2>&1
  echo "$V c2: $(grep 'policy [0-7] ' $OUT/w_$V.log | head -8 | awk '{printf "%d ", $9/1e6}') | $(tail -1 $OUT/w_$V.log | grep -o 'kernel.*')"
  GML_LIB=build/libgml_$V.so timeout 300 python tools/run_replay.py --workload c3 --reps 2 2>&1 | tail -1 | grep -o "kernel.*" | sed "s|^|$V c3: |"
 done
done
