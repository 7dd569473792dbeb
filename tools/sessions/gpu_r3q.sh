#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/b.log 2>&1; echo "build=$?"
for r in 1 2; do
  for E in "" "GML_NO_PERSIST=1"; do
    env $E GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 3 2>&1 | grep kernel | awk '{print $(NF-1)}' | tr '\n' ' ' | sed "s|^|c4 [$E]: |"; echo
  done
done
GML_C4_PER_GPU=512 timeout 900 python tools/split_check.py c4 2 2>&1 | grep -v Warn | tail -3
timeout 900 python -m pytest tests/test_split_gpu.py tests/test_parity_gpu.py -q -x -k "path or c4 or m4 or random_policy" > $OUT/pt.log 2>&1; echo "pytest=$?"; tail -2 $OUT/pt.log
