#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python tools/build_variants.py l1=GML_LAZY_PIN=1 l2=GML_LAZY_PIN=2 > $OUT/bv.log 2>&1; echo "build=$?"
for r in 1 2; do
 for V in l1 l2; do
  GML_LIB=build/libgml_$V.so GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 1 > $OUT/v_$V.log 2>&1
  echo "$V c2: $(grep 'policy [0-7] ' $OUT/v_$V.log | head -8 | awk '{printf "%d ", $9/1e6}') | $(tail -1 $OUT/v_$V.log | grep -o 'kernel.*')"
 done
done
