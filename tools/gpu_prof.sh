#!/bin/bash
# ncu --set full of K1 on a workload (optionally a policy subset); exports
# raw metrics + per-source-line hot spots to gpurun_out/.
# Usage (under gpurun): bash tools/gpu_prof.sh <tag> <workload> [policies]
set -u
TAG=$1; WL=$2; POL=${3:-}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ARGS="--workload $WL --reps 1"
[ -n "$POL" ] && ARGS="$ARGS --policies $POL"
timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
    -k regex:k_replay -c 12 -o /tmp/prof_$TAG python tools/run_replay.py $ARGS > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu=$?"
ncu -i /tmp/prof_$TAG.ncu-rep --page raw --csv > $OUT/raw_$TAG.csv 2>/dev/null
ncu -i /tmp/prof_$TAG.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_$TAG.csv 2>/dev/null
python tools/ncu_lines.py /tmp/src_$TAG.csv 80 > $OUT/hot_lines_$TAG.txt 2>&1
head -40 $OUT/hot_lines_$TAG.txt
