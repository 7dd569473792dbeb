#!/bin/bash
# Build, GPU tests, one bench line. Usage (under gpurun): bash tools/gpu_check.sh <tag> [pytest -k expr]
set -u
TAG=${1:-chk}; K=${2:-}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1; echo "build=$?"
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x -k "$K" > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?"
else
  timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?"
fi
tail -5 $OUT/pytest_gpu_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench=$?"; head -c 400 $OUT/bench_$TAG.json; echo
python - <<PY
import json
d=json.load(open("$OUT/bench_$TAG.json"))
print("C2", d["value"], d["ms_per_step"], "C4", d["secondary_c4"]["value"], d["secondary_c4"]["ms_per_step"])
for k,v in d["policies"].items(): print(k, {a: (round(b,4) if isinstance(b,float) else b) for a,b in v.items()})
PY
