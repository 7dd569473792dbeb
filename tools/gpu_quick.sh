#!/bin/bash
# Build, gpu tests, per-unit cycles (+ phases) on C2, one bench line.
# Usage (under gpurun): bash tools/gpu_quick.sh <tag> [notests] [nobench]
set -u
TAG=${1:-q}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.build_prof()" > $OUT/build_$TAG.log 2>&1; echo "build=$?"
if [[ " $* " != *" notests "* ]]; then
  timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?"; tail -3 $OUT/pytest_gpu_$TAG.log
fi
GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 1 > $OUT/cycles_c2_$TAG.log 2>&1; echo "cycles=$?"; tail -9 $OUT/cycles_c2_$TAG.log
GML_LIB=build/libgml_prof.so GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 1 > $OUT/phases_c2_$TAG.log 2>&1; echo "phases=$?"; tail -9 $OUT/phases_c2_$TAG.log
if [[ " $* " != *" nobench "* ]]; then
  timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench=$?"; head -c 600 $OUT/bench_$TAG.json; echo
  python -c "import json;d=json.load(open('$OUT/bench_$TAG.json'));s=d['secondary_c4'];print('C4',s['value'],s['ms_per_step'],s['roofline']['kernel_ms'])"
fi
