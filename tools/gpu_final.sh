#!/bin/bash
# Final check: full GPU suite + smoke, then the default bench line.
set -u
TAG=${1:-final}
OUT=gpurun_out; mkdir -p $OUT
bash tools/gpu_tests.sh $TAG
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench=$?"; head -c 400 $OUT/bench_$TAG.json; echo
