#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/b.log 2>&1; echo "build=$?"
for r in 1 2; do
 for L in paper_2401_08156_b200/libgml.so build/libgml_prev.so; do
  GML_LIB=$L GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 1 > $OUT/ab_$r.log 2>&1
  echo "$L c2: $(grep 'policy [0-7] ' $OUT/ab_$r.log | head -8 | awk '{printf "%.1f ", $9/1e6}') | $(tail -1 $OUT/ab_$r.log | grep -o 'kernel.*')"
 done
done
