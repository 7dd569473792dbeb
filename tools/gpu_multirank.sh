#!/bin/bash
# Exercise bench.py's N>1 path on a 1-GPU box: 2 ranks sharing cuda:0 over
# gloo (the driver's runs use one GPU per rank and NCCL), torchrun with one
# NCCL rank, and the reference arm under torchrun.
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
GML_SAME_DEVICE=1 GML_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 \
  > $OUT/bench_w2_gloo.json 2> $OUT/bench_w2_gloo.err; echo "w2=$?"; head -c 700 $OUT/bench_w2_gloo.json; echo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --no-secondary > $OUT/bench_w1_nccl.json 2> $OUT/bench_w1_nccl.err; echo "w1=$?"; head -c 300 $OUT/bench_w1_nccl.json; echo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > $OUT/bench_ref_w2.json 2> $OUT/bench_ref_w2.err; echo "ref=$?"; head -c 500 $OUT/bench_ref_w2.json; echo
