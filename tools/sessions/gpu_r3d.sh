#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/b.log 2>&1; echo "build=$?"
timeout 300 python tools/split_check.py c2 3 > $OUT/sc_c2.log 2>&1
timeout 300 python tools/split_check.py c3 3 > $OUT/sc_c3.log 2>&1
GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --workload c2 --reps 1 > $OUT/cyc_c2.log 2>&1
cat $OUT/sc_c2.log $OUT/sc_c3.log; tail -9 $OUT/cyc_c2.log
timeout 900 python -m pytest tests/test_split_gpu.py tests/test_parity_gpu.py -q -x -k "split or fuzz or invalid or overflow or c2 or c3 or fig or irregular or ragged or extreme" > $OUT/pt.log 2>&1; echo "pytest=$?"; tail -3 $OUT/pt.log
