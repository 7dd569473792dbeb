set -u
python -c "import paper_2401_08156_b200.gml as g" 2>&1 | tail -1
for r in 1 2 3; do for V in oldb3f cur ev0 fz1 fz2 fz1ev0; do
  GML_LIB=build/libgml_$V.so GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 2 2>&1 | tail -1 | sed "s|^.*wall, |$V r$r: |"
done; done
