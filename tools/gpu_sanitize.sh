#!/bin/bash
# compute-sanitizer over K0/K1 (shared-memory and global-memory arenas).
# Usage (under gpurun): bash tools/gpu_sanitize.sh <tag>
set -u
TAG=${1:-san}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1; echo "build=$?"
# initcheck runs on the build that zeroes the BFC free lists at init
# (GML_FL_ZERO=1): the product build's best-fit vectors read never-written
# slots outside a pool and mask them off, which initcheck would report
python tools/build_variants.py "flz=GML_FL_ZERO=1" >> $OUT/build_$TAG.log 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
for mode in smem global throughput; do
  unset GML_FORCE_GLOBAL GML_SAN_THROUGHPUT
  [ $mode = global ] && export GML_FORCE_GLOBAL=1
  [ $mode = throughput ] && export GML_SAN_THROUGHPUT=1
  for tool in memcheck racecheck synccheck initcheck; do
    lib=paper_2401_08156_b200/libgml.so; [ $tool = initcheck ] && lib=build/libgml_flz.so
    GML_LIB=$lib timeout 1500 $CS --tool $tool --error-exitcode 9 --print-limit 20 \
        python tools/sanitize_replay.py > $OUT/sanitize_${TAG}_${mode}_${tool}.log 2>&1
    echo "$mode $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|parity' $OUT/sanitize_${TAG}_${mode}_${tool}.log | tr '\n' ' ')"
  done
done
