set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_r2d.log 2>&1; echo build=$?
for pad in 0 120000 0 120000; do
  GML_GLOBAL_SMEM_PAD=$pad GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 3 2>&1 | tail -1 | sed "s|^|pad=$pad c4: |"
done
python tools/build_variants.py "u2m3=GML_SHIFT_U=2,GML_GLOBAL_MINB=3" "u1m3=GML_SHIFT_U=1,GML_GLOBAL_MINB=3" "u2=GML_SHIFT_U=2" >> $OUT/build_r2d.log 2>&1
for r in 1 2; do for V in u2m3 u1m3 u2; do
  GML_LIB=build/libgml_$V.so GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 3 2>&1 | tail -1 | sed "s|^|$V c4: |"
done; done
timeout 900 python bench.py > $OUT/bench_r2d.json 2> $OUT/bench_r2d.err; echo "bench=$?"
python - <<PY
import json
d=json.load(open("$OUT/bench_r2d.json"))
print("C2", d["value"], d["ms_per_step"], "cold", d["cold"]["value"], "cpu", d["cpu_baseline"]["value"])
s=d["secondary_c4"]; print("C4", s["value"], s["ms_per_step"], "cold", s["cold"]["value"], s["cold"]["ms_per_step"])
print("c5", json.dumps(d["c5_live"])[:600])
PY
bash tools/gpu_multirank.sh
