#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.build_prof()" > $OUT/b.log 2>&1; echo "build=$?"
GML_LIB=build/libgml_prof.so GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --workload c2 --reps 1 > $OUT/phases_c2_split.log 2>&1
tail -9 $OUT/phases_c2_split.log
