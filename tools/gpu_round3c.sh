#!/bin/bash
# Final-build session: bench line, launch list, C2 full capture (traffic, kernels), C2 chain profile.
set -u
TAG=${1:-r3c}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1; echo "build=$?"
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench=$?"; head -c 300 $OUT/bench_$TAG.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/bench_ncu_$TAG.log 2>&1; echo "ncu_launches=$?"
timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
    -k regex:"k_replay|k_ledger|k_merge|k_max_slot" -c 16 -o /tmp/prof_c2 python tools/run_replay.py --workload c2 --reps 1 > $OUT/ncu_full_c2_$TAG.log 2>&1; echo "ncu_c2=$?"
ncu -i /tmp/prof_c2.ncu-rep --page raw --csv > $OUT/raw_c2_$TAG.csv 2>/dev/null
python tools/ncu_kernels.py $OUT/raw_c2_$TAG.csv > $OUT/ncu_kernels_c2_$TAG.json 2>&1
python tools/ncu_traffic.py $OUT/raw_c2_$TAG.csv c2 $OUT/ncu_c2_traffic.json
bash tools/gpu_units.sh $TAG > $OUT/units_$TAG.log 2>&1; echo "units=$?"
