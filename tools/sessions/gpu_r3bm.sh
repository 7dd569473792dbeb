#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python tools/build_variants.py bm0=GML_PATH_BM_SMEM=0 > $OUT/bv.log 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/b.log 2>&1; echo "build=$?"
for r in 1 2; do
 for L in paper_2401_08156_b200/libgml.so build/libgml_bm0.so; do
  GML_LIB=$L GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 3 2>&1 | grep kernel | awk '{print $(NF-1)}' | tr '\n' ' ' | sed "s|^|$L c4: |"; echo
 done
done
timeout 1200 python -m pytest tests/test_split_gpu.py tests/test_parity_gpu.py -q -x -k "path or c4 or m4 or random_policy or fuzz" > $OUT/pt.log 2>&1; echo "pytest=$?"; tail -1 $OUT/pt.log
