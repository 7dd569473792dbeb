#!/bin/bash
# A/B timing of two builds on C4 and C2 (run_replay, interleaved reps).
# Usage: bash tools/gpu_ab.sh <flagsB>   (B = current sources built with extra -D flags)
set -u
OUT=gpurun_out; mkdir -p $OUT
FLAGS=${1:-}
python - <<PY > $OUT/ab_build.log 2>&1
import __graft_entry__ as g
from pathlib import Path
g.build()
g.build(extra_flags=tuple("$FLAGS".split()), lib=Path("build/libgml_b.so"))
PY
echo "build=$?"
for r in 1 2; do
 for L in paper_2401_08156_b200/libgml.so build/libgml_b.so; do
  GML_LIB=$L GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 3 2>&1 | tail -2 | sed "s|^|$L c4: |"
  GML_LIB=$L timeout 600 python tools/run_replay.py --workload c2 --reps 2 2>&1 | tail -1 | sed "s|^|$L c2: |"
 done
done
