#!/bin/bash
# compute-sanitizer over K0/K1 (shared-memory and global-memory arenas).
# Usage (under gpurun): bash tools/gpu_sanitize.sh <tag>
set -u
TAG=${1:-san}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1; echo "build=$?"
CS=/usr/local/cuda/bin/compute-sanitizer
for mode in smem global; do
  if [ $mode = global ]; then export GML_FORCE_GLOBAL=1; else unset GML_FORCE_GLOBAL; fi
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 1500 $CS --tool $tool --error-exitcode 9 --print-limit 20 \
        python tools/sanitize_replay.py > $OUT/sanitize_${TAG}_${mode}_${tool}.log 2>&1
    echo "$mode $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|parity' $OUT/sanitize_${TAG}_${mode}_${tool}.log | tr '\n' ' ')"
  done
done
