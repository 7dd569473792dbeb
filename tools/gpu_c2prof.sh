#!/bin/bash
# C2 per-unit cycles + phases + ncu source-level hot lines (both rankings).
# Usage (under gpurun): bash tools/gpu_c2prof.sh <tag> [policies]
set -u
TAG=$1; POL=${2:-}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.build_prof()" > $OUT/build_$TAG.log 2>&1; echo "build=$?"
GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 1 > $OUT/cycles_c2_$TAG.log 2>&1; tail -9 $OUT/cycles_c2_$TAG.log
GML_LIB=build/libgml_prof.so GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 1 > $OUT/phases_c2_$TAG.log 2>&1; tail -9 $OUT/phases_c2_$TAG.log
bash tools/gpu_prof.sh $TAG c2 $POL > /dev/null 2>&1; echo "prof=$?"
