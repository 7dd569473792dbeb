#!/bin/bash
# A/B: ledger poll interval (C2 per-warp cycles + kernel ms)
set -u
OUT=gpurun_out; mkdir -p $OUT
python tools/build_variants.py base= ns20k=GML_LEDGER_NS=20000 ns200k=GML_LEDGER_NS=200000 > $OUT/bv.log 2>&1; echo "build=$?"
for r in 1 2; do
 for V in base ns20k ns200k; do
  GML_LIB=build/libgml_$V.so GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 1 > $OUT/ld_${V}_$r.log 2>&1
  echo "$V c2: $(grep 'policy 3 ' $OUT/ld_${V}_$r.log | awk '{print $9, $17, $18, $19}') | $(tail -1 $OUT/ld_${V}_$r.log | grep -o 'kernel.*')"
 done
done
GML_SPLIT_VMM_ONLY=1 GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 1 2>&1 | grep 'policy 3 ' | awk '{print "vmm-only", $9, $17}'
