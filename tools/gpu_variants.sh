#!/bin/bash
# Per-unit cycles on C2 (and C4 kernel time) for prebuilt library variants
# build/libgml_<name>.so (built here with tools/build_variants.py).
# Usage (under gpurun): bash tools/gpu_variants.sh <tag> <name>...
set -u
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
for r in 1 2; do
  for V in "$@"; do
    GML_LIB=build/libgml_$V.so GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 1 > $OUT/var_${TAG}_${V}_$r.log 2>&1
    echo "$V run$r: $(grep -o 'cycles [0-9]*' $OUT/var_${TAG}_${V}_$r.log | awk '{printf "%d ", $2/1e6}') | $(tail -1 $OUT/var_${TAG}_${V}_$r.log | grep -o 'kernel.*')"
  done
done
if [ -n "${C4:-}" ]; then
  for V in "$@"; do
    GML_LIB=build/libgml_$V.so GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 3 2>&1 | tail -1 | sed "s|^|$V c4: |"
  done
fi
