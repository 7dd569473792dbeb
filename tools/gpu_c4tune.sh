#!/bin/bash
# C4 occupancy experiment: K1 global-arena instances at 2 / 3 CTAs per SM.
set -u
OUT=gpurun_out; mkdir -p $OUT
python - <<'PY' > $OUT/c4tune_build.log 2>&1
import __graft_entry__ as g
from pathlib import Path
g.build()
for m in (3, 4):
    g.build(extra_flags=(f"-DGML_GLOBAL_MINB={m}",), lib=Path(f"build/libgml_minb{m}.so"))
PY
echo "build=$?"; grep -c "spill" $OUT/c4tune_build.log
for L in paper_2401_08156_b200/libgml.so build/libgml_minb3.so build/libgml_minb4.so; do
  GML_LIB=$L GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 3 2>&1 | tail -3 | sed "s|^|$L: |"
done
