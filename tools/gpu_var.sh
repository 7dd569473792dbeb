#!/bin/bash
# Build library variants on the box and time them on C4 and C2 (interleaved).
# Usage (under gpurun): bash tools/gpu_var.sh <tag> name=FLAGS ...   (name=base: no extra flags)
set -u
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1
names=()
for spec in "$@"; do
  names+=("${spec%%=*}")
  python tools/build_variants.py "$spec" >> $OUT/build_$TAG.log 2>&1 || echo "build $spec failed"
done
for r in 1 2; do
  for V in "${names[@]}"; do
    L=build/libgml_$V.so
    GML_LIB=$L GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 3 2>&1 | tail -1 | sed "s|^|$V c4 r$r: |"
    GML_LIB=$L GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 1 > $OUT/var_${TAG}_${V}_$r.log 2>&1
    echo "$V c2 r$r: $(grep -o 'cycles [0-9]*' $OUT/var_${TAG}_${V}_$r.log | awk '{printf "%d ", $2/1e6}') | $(tail -1 $OUT/var_${TAG}_${V}_$r.log | grep -o 'kernel.*')"
  done
done
