#!/bin/bash
# Deployment-mode measurements: live allocator latency (C5) and a PyTorch
# training run under the default allocator vs GMLake (f3), step times.
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python tools/live_latency.py --iters 4 > $OUT/live_latency.json 2> $OUT/live_latency.err; echo "live=$?"
for m in "" "--gml"; do
  timeout 900 python tests/workloads/torch_train.py --steps 15 $m > $OUT/train$m.json 2> $OUT/train$m.err; echo "train$m=$?"
done
timeout 900 python tests/workloads/torch_train.py --steps 15 --gml --limit-mib 2 > $OUT/train_gml_lim2.json 2> $OUT/train_gml_lim2.err; echo "lim2=$?"
