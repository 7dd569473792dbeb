set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import paper_2401_08156_b200.gml as g" 2>&1 | tail -1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
for r in 1 2 3; do for V in oldb3f cur; do
  for c in tight cold; do
    GML_LIB=build/libgml_$V.so GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 2 --caps $c 2>&1 | tail -1 | sed "s|^|$V $c c4 r$r: |"
  done
done; done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
