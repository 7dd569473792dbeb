#!/bin/bash
# A/B of Engine::free_run variants (GML_FREE_RUN=0 off, 1 distributed intervals, 2 per-lane intervals)
set -u
OUT=gpurun_out; mkdir -p $OUT
python tools/build_variants.py fr0=GML_FREE_RUN=0 fr1=GML_FREE_RUN=1 fr2=GML_FREE_RUN=2 > $OUT/bv.log 2>&1; echo "build=$?"
for r in 1 2; do
 for V in fr0 fr1 fr2; do
  GML_LIB=build/libgml_$V.so GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 1 > $OUT/fr_${V}_$r.log 2>&1
  echo "$V c2: $(grep -o 'phases [0-9]*' $OUT/fr_${V}_$r.log | awk '{printf "%d ", $2/1e6}') | $(tail -1 $OUT/fr_${V}_$r.log | grep -o 'kernel.*')"
  GML_LIB=build/libgml_$V.so GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 3 2>&1 | tail -1 | sed "s|^|$V c4: |"
  GML_NO_SPLIT=1 GML_LIB=build/libgml_$V.so timeout 300 python tools/run_replay.py --workload c3 --reps 2 2>&1 | tail -1 | sed "s|^|$V c3 serial: |"
 done
done
