#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/b.log 2>&1; echo "build=$?"
GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 1 > $OUT/y.log 2>&1
echo "c2: $(grep 'policy [0-7] ' $OUT/y.log | head -8 | awk '{printf "%.1f ", $9/1e6}') | $(tail -1 $OUT/y.log | grep -o 'kernel.*')"
timeout 300 python tools/run_replay.py --workload c3 --reps 2 2>&1 | tail -1 | grep -o "kernel.*" | sed "s|^|c3: |"
GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 3 2>&1 | grep kernel | awk '{print $(NF-1)}' | tr '\n' ' ' | sed "s|^|c4: |"; echo
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pt.log 2>&1; echo "pytest=$?"; tail -1 $OUT/pt.log
