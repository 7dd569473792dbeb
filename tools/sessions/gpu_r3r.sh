#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/b.log 2>&1; echo "build=$?"
for i in 1 2 3; do
  timeout 900 python -m pytest tests/test_split_gpu.py -q -x -k "path" > $OUT/pt_$i.log 2>&1; echo "run$i=$? $(tail -1 $OUT/pt_$i.log)"
done
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "m4 or m5 or random_policy or c4 or fuzz" > $OUT/pt_p.log 2>&1; echo "parity=$? $(tail -1 $OUT/pt_p.log)"
GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 3 2>&1 | grep kernel | awk '{print $(NF-1)}' | tr '\n' ' ' | sed "s|^|c4: |"; echo
