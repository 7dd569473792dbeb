#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python tools/build_variants.py pm4=GML_PATH_MINB=4 > $OUT/bv.log 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/b.log 2>&1; echo "build=$?"
timeout 900 python -m pytest tests/test_split_gpu.py -q -x > $OUT/pt_split.log 2>&1; echo "pytest_split=$?"; tail -2 $OUT/pt_split.log
for r in 1 2; do
 for L in paper_2401_08156_b200/libgml.so build/libgml_pm4.so; do
  GML_LIB=$L GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 3 2>&1 | grep kernel | awk '{print $(NF-1)}' | tr '\n' ' ' | sed "s|^|$L c4: |"; echo
 done
done
python - <<'PY'
import os, sys
sys.path.insert(0, '.')
os.environ["GML_C4_PER_GPU"] = "512"
import numpy as np, torch, bench
from paper_2401_08156_b200 import replay as R, gml
W = bench.Workload("c4", 1)
tr = W.load(list(range(W.n)))
b = R.upload(tr, "cuda:0")
caps = np.zeros((len(tr) * 8, 4), dtype=np.uint32)
R.run(b, W.pols, caps=caps); R.run(b, W.pols, caps=caps)
print("c4 split count (done, reruns):", gml.gml_last_split_count(), "launches", gml.gml_last_launch_count(), "kernel ms", gml.gml_last_kernel_ms())
PY
