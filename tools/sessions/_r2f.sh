set -u
OUT=gpurun_out; mkdir -p $OUT
bash tools/gpu_tests.sh r2f
for r in 1 2; do
  for c in tight cold; do
    GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 2 --caps $c 2>&1 | tail -1 | sed "s|^|caps=$c c4: |"
    GML_ONE_LAUNCH=1 GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 2 --caps $c 2>&1 | tail -1 | sed "s|^|one caps=$c c4: |"
  done
done
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool racecheck --error-exitcode 9 --print-limit 20 python tools/sanitize_replay.py > $OUT/sanitize_r2f_smem_racecheck.log 2>&1; echo "racecheck rc=$? $(grep -E 'SUMMARY' $OUT/sanitize_r2f_smem_racecheck.log)"
GML_FORCE_GLOBAL=1 timeout 1500 $CS --tool initcheck --error-exitcode 9 --print-limit 20 python tools/sanitize_replay.py > $OUT/sanitize_r2f_global_initcheck.log 2>&1; echo "initcheck rc=$? $(grep -E 'SUMMARY' $OUT/sanitize_r2f_global_initcheck.log)"
timeout 900 python bench.py > $OUT/bench_r2f.json 2> $OUT/bench_r2f.err; echo "bench=$?"
python - <<PY
import json
d=json.load(open("$OUT/bench_r2f.json"))
print("C2", d["value"], d["ms_per_step"], "cold", d["cold"]["value"], "cpu", d["cpu_baseline"]["value"])
s=d["secondary_c4"]; print("C4", s["value"], s["ms_per_step"], "cold", s["cold"]["value"], s["cold"]["ms_per_step"], "launches", s["gpu_launches"])
print("c5 bw", d["c5_live"]["stream_copy_gbs"])
PY
