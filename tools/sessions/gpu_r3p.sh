#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/b.log 2>&1; echo "build=$?"
for r in 1 2; do
 for L in paper_2401_08156_b200/libgml.so build/libgml_prev.so; do
  GML_LIB=$L GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 1 > $OUT/p_$r.log 2>&1
  echo "$L c2: $(grep 'policy [2-7] ' $OUT/p_$r.log | awk '{printf "%d ", $9/1e6}') | $(tail -1 $OUT/p_$r.log | grep -o 'kernel.*')"
  GML_LIB=$L timeout 300 python tools/run_replay.py --workload c3 --reps 2 2>&1 | tail -1 | grep -o 'kernel.*' | sed "s|^|$L c3: |"
 done
done
timeout 900 python tools/split_check.py c2 1 2>&1 | tail -3
timeout 900 python -m pytest tests/test_split_gpu.py tests/test_parity_gpu.py -q -x -k "split or path or c2 or c3 or overflow or fuzz or fig or irregular" > $OUT/pt.log 2>&1; echo "pytest=$?"; tail -2 $OUT/pt.log
