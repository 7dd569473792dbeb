#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/b.log 2>&1; echo "build=$?"
for r in 1 2; do
 for E in "" "GML_NO_PRIO=1"; do
  env $E GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 3 2>&1 | grep kernel | awk '{print $(NF-1)}' | tr '\n' ' ' | sed "s|^|c4 [$E]: |"; echo
 done
done
