set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_r2k.log 2>&1; echo build=$?
cp paper_2401_08156_b200/libgml.so build/libgml_base.so
python tools/build_variants.py "cn=GML_COLD_NOINL" "cn3=GML_COLD_NOINL,GML_GLOBAL_MINB=3" "cn3w2=GML_COLD_NOINL,GML_GLOBAL_WPC=2,GML_GLOBAL_MINB=6" >> $OUT/build_r2k.log 2>&1
grep -E "registers|stack" $OUT/build_r2k.log | sort | uniq -c | sort -rn | head -5
for r in 1 2 3; do for V in base cn cn3 cn3w2; do
  GML_LIB=build/libgml_$V.so GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 2 2>&1 | tail -1 | sed "s|^|$V c4 r$r: |"
done; done
for V in base cn; do
  GML_LIB=build/libgml_$V.so GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 1 > $OUT/var_r2k_${V}.log 2>&1
  echo "$V c2: $(grep -o 'cycles [0-9]*' $OUT/var_r2k_${V}.log | awk '{printf "%d ", $2/1e6}') | $(tail -1 $OUT/var_r2k_${V}.log | grep -o 'kernel.*')"
done
