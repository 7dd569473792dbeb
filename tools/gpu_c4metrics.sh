#!/bin/bash
# C4: targeted ncu metrics of every kernel of one gml_replay (application
# replay, a handful of passes instead of --set full's ~40):
# DRAM bytes, warp instructions, achieved occupancy, issue activity, L1/L2 hit rates.
# Usage (under gpurun): bash tools/gpu_c4metrics.sh <tag>
set -u
TAG=${1:-c4m}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
M=$M,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
M=$M,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,launch__registers_per_thread,launch__occupancy_limit_registers
M=$M,sm__maximum_warps_per_active_cycle_pct,launch__grid_size,launch__block_size
GML_C4_PER_GPU=512 timeout 1500 ncu --metrics $M --clock-control none --replay-mode application --nvtx --nvtx-include "timed/" \
    -k regex:"k_replay|k_ledger|k_merge|k_max_slot" -c 16 -o /tmp/c4m_$TAG python tools/run_replay.py --workload c4 --reps 1 > $OUT/ncu_c4m_$TAG.log 2>&1; echo "ncu=$?"
ncu -i /tmp/c4m_$TAG.ncu-rep --page raw --csv > $OUT/raw_c4m_$TAG.csv 2>/dev/null
python tools/ncu_traffic.py $OUT/raw_c4m_$TAG.csv c4 $OUT/ncu_c4_traffic.json
python tools/ncu_kernels.py $OUT/raw_c4m_$TAG.csv > $OUT/ncu_kernels_c4m_$TAG.json 2>&1
