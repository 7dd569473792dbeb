#!/bin/bash
set -u
POL=${1:-3}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/b.log 2>&1
GML_SPLIT_VMM_ONLY=1 timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
    -k regex:k_replay_split -c 1 -o /tmp/prof_v3 python tools/run_replay.py --workload c2 --reps 1 --policies $POL > $OUT/ncu_v3.log 2>&1; echo "ncu=$?"
ncu -i /tmp/prof_v3.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_v3.csv 2>/dev/null
python tools/ncu_lines.py /tmp/src_v3.csv 70 > $OUT/hot_lines_c2_v${POL}_vmmwarp_r3.txt 2>&1
ncu -i /tmp/prof_v3.ncu-rep --page raw --csv > $OUT/raw_v3.csv 2>/dev/null
head -75 $OUT/hot_lines_c2_v${POL}_vmmwarp_r3.txt
