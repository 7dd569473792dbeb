set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_r2e.log 2>&1; echo build=$?
for r in 1 2; do
  for c in tight cold 4000,2000,8000,4000 2000,1000,4000,2000; do
    GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 2 --caps $c 2>&1 | tail -1 | sed "s|^|caps=$c c4: |"
  done
  GML_FORCE_SMEM=1 GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 2 2>&1 | tail -1 | sed "s|^|smem c4: |"
done
bash tools/gpu_sanitize.sh r2e
