#!/bin/bash
# Per-unit chain profile of C2: each policy variant replayed alone under ncu
# (instructions, cycles, stall reasons of its single-warp unit; a GMLake
# unit is a split unit whose VMM warp runs alone, GML_SPLIT_VMM_ONLY) ->
# gpurun_out/ncu_c2_units.json. Usage (under gpurun): bash tools/gpu_units.sh <tag>
set -u
TAG=${1:-u}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1
M=smsp__inst_executed.sum,sm__cycles_elapsed.max,gpu__time_duration.sum
for s in wait branch_resolving selected short_scoreboard no_instructions long_scoreboard mio_throttle misc dispatch_stall barrier membar; do
  M=$M,smsp__pcsamp_warps_issue_stalled_$s
done
for pol in 0 1 2 3 4 5 6 7; do
  GML_SPLIT_VMM_ONLY=1 timeout 600 ncu --metrics $M --clock-control none --nvtx --nvtx-include "timed/" -k regex:k_replay --csv \
     python tools/run_replay.py --workload c2 --reps 1 --policies $pol > $OUT/units_${TAG}_v$pol.csv 2> $OUT/units_${TAG}_v$pol.err
  echo "v$pol rc=$?"
done
python tools/ncu_units.py $OUT/units_${TAG}_v{0,1,2,3,4,5,6,7}.csv > $OUT/ncu_c2_units.json; cat $OUT/ncu_c2_units.json | head -40
