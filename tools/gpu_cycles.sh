#!/bin/bash
# Per-unit cycles + phase counters on a workload, both executors.
# Usage (under gpurun): bash tools/gpu_cycles.sh <tag> [workload]
set -u
TAG=${1:-d}; WL=${2:-c2}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.build_prof()" > $OUT/build_$TAG.log 2>&1; echo "build=$?"
for MODE in warp cta; do
  GML_MODE=$MODE GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --workload $WL --reps 1 > $OUT/cycles_${WL}_${MODE}_$TAG.log 2>&1; echo "cycles_$MODE=$?"; tail -9 $OUT/cycles_${WL}_${MODE}_$TAG.log
  GML_MODE=$MODE GML_LIB=build/libgml_prof.so GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --workload $WL --reps 1 > $OUT/phases_${WL}_${MODE}_$TAG.log 2>&1; echo "phases_$MODE=$?"; tail -9 $OUT/phases_${WL}_${MODE}_$TAG.log
done
