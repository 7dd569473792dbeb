#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python tools/build_variants.py base= bfc5=GML_BFC_MINB=5 > $OUT/bv.log 2>&1; echo "build=$?"
for r in 1 2; do
 for V in base bfc5; do
  GML_LIB=build/libgml_$V.so GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 3 2>&1 | grep kernel | awk '{print $(NF-1)}' | tr '\n' ' ' | sed "s|^|$V c4: |"; echo
 done
done
for V in base bfc5; do GML_LIB=build/libgml_$V.so timeout 300 python tools/run_replay.py --reps 2 2>&1 | tail -1 | grep -o "kernel.*" | sed "s|^|$V c2: |"; done
