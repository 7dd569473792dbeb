#!/bin/bash
# A/B of path-unit variants on C4 (kernel ms)
set -u
OUT=gpurun_out; mkdir -p $OUT
python tools/build_variants.py base= pm3=GML_PATH_MINB=3 pfr=GML_PATH_FREE_RUN=1 > $OUT/bv.log 2>&1; echo "build=$?"
for r in 1 2; do
 for V in base pm3 pfr; do
  GML_LIB=build/libgml_$V.so GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 3 2>&1 | grep kernel | awk '{print $(NF-1)}' | tr '\n' ' ' | sed "s|^|$V c4: |"; echo
 done
done
GML_NO_SPLIT=1 GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 3 2>&1 | grep kernel | awk '{print $(NF-1)}' | tr '\n' ' ' | sed "s|^|serial c4: |"; echo
