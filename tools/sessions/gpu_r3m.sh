#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
git_stash=0
python tools/build_variants.py nofr=GML_FREE_RUN=0 > $OUT/bv.log 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/b.log 2>&1; echo "build=$?"
for r in 1 2; do
 for L in paper_2401_08156_b200/libgml.so build/libgml_nofr.so; do
  GML_LIB=$L GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 1 > $OUT/m_$r.log 2>&1
  echo "$L: $(grep 'policy 3 ' $OUT/m_$r.log | head -1 | awk '{print $9}') $(tail -1 $OUT/m_$r.log | grep -o 'kernel.*')"
 done
done
