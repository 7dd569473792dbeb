#!/bin/bash
# GPU session for the NEXT rows: their tests, VMM latency (f2), convergence + grid (f4).
set -u
TAG=${1:-n}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1; echo "build=$?"
timeout 1500 python -m pytest tests/test_torch_backend_gpu.py tests/test_parity_gpu.py -m gpu -q -x -k "torch or snapshot or timeline or convergence" -s > $OUT/pytest_next_$TAG.log 2>&1; echo "pytest=$?"; tail -5 $OUT/pytest_next_$TAG.log
timeout 600 python tools/vmm_latency.py --reps 5 > $OUT/vmm_latency_$TAG.json 2> $OUT/vmm_latency_$TAG.err; echo "vmm=$?"
timeout 900 python tools/convergence.py > $OUT/convergence_$TAG.json 2> $OUT/convergence_$TAG.err; echo "conv=$?"
