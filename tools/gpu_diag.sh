#!/bin/bash
# Quick GPU diagnosis: gpu tests, per-unit cycles and phase counters on C2.
# Usage (under gpurun): bash tools/gpu_diag.sh <tag> [skip_tests]
set -u
TAG=${1:-d}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.build_prof()" > $OUT/build_$TAG.log 2>&1; echo "build=$?"
if [ "${2:-}" != "skip_tests" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?"; tail -2 $OUT/pytest_gpu_$TAG.log
fi
GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 2 > $OUT/cycles_c2_$TAG.log 2>&1; echo "cycles=$?"; tail -12 $OUT/cycles_c2_$TAG.log
GML_LIB=build/libgml_prof.so GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 1 > $OUT/phases_c2_$TAG.log 2>&1; echo "phases=$?"; tail -10 $OUT/phases_c2_$TAG.log
