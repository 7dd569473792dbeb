#!/bin/bash
# One GPU session: tests, smoke, bench, launch list, full profile of K1.
# Usage (under gpurun): bash tools/gpu_round.sh <tag>
set -u
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?"; tail -2 $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke=$?"; tail -1 $OUT/smoke_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench=$?"; tail -c 1500 $OUT/bench_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-secondary > $OUT/bench_ncu_$TAG.log 2>&1; echo "ncu_launches=$?"
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:k_replay -c 8 \
    -o $OUT/prof_c2_$TAG python tools/run_replay.py --reps 1 > $OUT/ncu_full_c2_$TAG.log 2>&1; echo "ncu_full_c2=$?"
GML_C4_PER_GPU=512 timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:k_replay -c 12 \
    -o $OUT/prof_c4_$TAG python tools/run_replay.py --workload c4 --reps 1 > $OUT/ncu_full_c4_$TAG.log 2>&1; echo "ncu_full_c4=$?"
