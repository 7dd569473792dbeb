#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/b.log 2>&1; echo "build=$?"
GML_C4_PER_GPU=512 timeout 600 python tools/split_check.py c4 3 > $OUT/sc_c4.log 2>&1; echo "sc_c4=$?"
grep -v Warn $OUT/sc_c4.log | tail -12
timeout 1500 python -m pytest tests/test_parity_gpu.py -q -x -k "c4_bench or m4 or random_policy or fuzz or overflow or global_arena" > $OUT/pt.log 2>&1; echo "pytest=$?"; tail -3 $OUT/pt.log
