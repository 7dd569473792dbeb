#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/b.log 2>&1; echo "build=$?"
GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 1 > $OUT/x.log 2>&1
echo "c2: $(grep 'policy [0-7] ' $OUT/x.log | head -8 | awk '{printf "%d ", $9/1e6}') | $(tail -1 $OUT/x.log | grep -o 'kernel.*')"
timeout 1800 python -m pytest tests/test_split_gpu.py tests/test_parity_gpu.py -q -x > $OUT/pt.log 2>&1; echo "pytest=$?"; tail -1 $OUT/pt.log
