#!/bin/bash
set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/b.log 2>&1; echo "build=$?"
cp paper_2401_08156_b200/libgml.so build/libgml_new.so
git_rev=$(cat .git_prev_rev 2>/dev/null)
for r in 1 2; do
 for L in build/libgml_new.so build/libgml_prev.so; do
  [ -f $L ] || continue
  GML_LIB=$L GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 3 2>&1 | grep kernel | awk '{print $(NF-1)}' | tr '\n' ' ' | sed "s|^|$L c4: |"; echo
 done
done
timeout 900 python -m pytest tests/test_split_gpu.py -q -x > $OUT/pt_split.log 2>&1; echo "pytest_split=$?"; tail -2 $OUT/pt_split.log
