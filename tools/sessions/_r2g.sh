set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.build_prof()" > $OUT/build_r2g.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "c4_bench or global_arena or overflow or tiny_corpus_m4" > $OUT/pytest_gpu_r2g.log 2>&1; echo "pytest=$?"; tail -1 $OUT/pytest_gpu_r2g.log
for r in 1 2; do
  for c in tight cold; do
    GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 2 --caps $c 2>&1 | tail -1 | sed "s|^|caps=$c c4: |"
  done
done
GML_LIB=build/libgml_prof.so GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 1 > $OUT/phases_c2_r2g.log 2>&1; echo "phases=$?"; grep gml-unit $OUT/phases_c2_r2g.log | tail -8
GML_UNIT_CYCLES=1 timeout 300 python tools/run_replay.py --reps 1 > $OUT/cycles_c2_r2g.log 2>&1; grep gml-unit $OUT/cycles_c2_r2g.log | tail -8 | awk '{print $4, $8}'
timeout 900 python bench.py > $OUT/bench_r2g.json 2> $OUT/bench_r2g.err; echo "bench=$?"
python - <<PY
import json
d=json.load(open("$OUT/bench_r2g.json"))
print("C2", d["value"], d["ms_per_step"], "cold", d["cold"]["value"], "cpu", d["cpu_baseline"]["value"])
s=d["secondary_c4"]; print("C4", s["value"], s["ms_per_step"], "cold", s["cold"]["value"], s["cold"]["ms_per_step"], "launches", s["gpu_launches"])
PY
