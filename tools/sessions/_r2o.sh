set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import paper_2401_08156_b200.gml as g" 2>&1 | tail -1
for r in 1 2 3; do for V in oldb3f cur fz1 fz2; do
  GML_LIB=build/libgml_$V.so GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 2 2>&1 | tail -1 | sed "s|^.*wall, |$V r$r: |"
done; done
GML_LIB=build/libgml_cur.so GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 1 > $OUT/var_r2o_cur.log 2>&1
echo "cur c2: $(grep -o 'cycles [0-9]*' $OUT/var_r2o_cur.log | awk '{printf "%d ", $2/1e6}') | $(tail -1 $OUT/var_r2o_cur.log | grep -o 'kernel.*')"
CS=/usr/local/cuda/bin/compute-sanitizer
export GML_LIB=build/libgml_cur.so
timeout 1500 $CS --tool initcheck --error-exitcode 9 --print-limit 20 python tools/sanitize_replay.py > $OUT/sanitize_r2o_smem_initcheck.log 2>&1; echo "smem initcheck rc=$? $(grep -E 'SUMMARY' $OUT/sanitize_r2o_smem_initcheck.log)"
GML_FORCE_GLOBAL=1 timeout 1500 $CS --tool initcheck --error-exitcode 9 --print-limit 20 python tools/sanitize_replay.py > $OUT/sanitize_r2o_global_initcheck.log 2>&1; echo "global initcheck rc=$? $(grep -E 'SUMMARY' $OUT/sanitize_r2o_global_initcheck.log)"
