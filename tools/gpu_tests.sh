#!/bin/bash
# Build + the whole GPU suite (no -x) + smoke. Usage (under gpurun): bash tools/gpu_tests.sh <tag> [pytest -k expr]
set -u
TAG=${1:-t}; K=${2:-}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1; echo "build=$?"
if [ -n "$K" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -k "$K" > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?"
else
  timeout 2400 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest=$?"
fi
grep -E "passed|failed|FAILED|Error" $OUT/pytest_gpu_$TAG.log | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke=$?"; tail -1 $OUT/smoke_$TAG.log
