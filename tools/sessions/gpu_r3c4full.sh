#!/bin/bash
# ncu --set full of the C4 top kernel (VMM path units), on a 128-trace C4 batch (kernel replay)
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
GML_C4_PER_GPU=128 timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
    -k regex:"k_replay_path" -c 1 -o /tmp/prof_c4p python tools/run_replay.py --workload c4 --reps 1 > $OUT/ncu_c4p.log 2>&1; echo "ncu=$?"
ncu -i /tmp/prof_c4p.ncu-rep --page raw --csv > $OUT/raw_c4p.csv 2>/dev/null
ncu -i /tmp/prof_c4p.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_c4p.csv 2>/dev/null
python tools/ncu_lines.py /tmp/src_c4p.csv 50 > $OUT/hot_lines_c4_vmmpath_r3.txt 2>&1
python tools/ncu_kernels.py $OUT/raw_c4p.csv > $OUT/ncu_kernels_c4p_r3.json 2>&1
head -30 $OUT/hot_lines_c4_vmmpath_r3.txt
