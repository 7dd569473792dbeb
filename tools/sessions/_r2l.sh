set -u
OUT=gpurun_out; mkdir -p $OUT
bash tools/gpu_tests.sh r2l
timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:k_replay -c 12 \
   --replay-mode application -o /tmp/prof_c4 python tools/run_replay.py --workload c4 --reps 1 > $OUT/ncu_full_c4_r2l.log 2>&1; echo "ncu_c4=$?"
ncu -i /tmp/prof_c4.ncu-rep --page raw --csv > $OUT/raw_c4_r2l.csv 2>/dev/null
ncu -i /tmp/prof_c4.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_c4.csv 2>/dev/null
python tools/ncu_lines.py /tmp/src_c4.csv 60 > $OUT/hot_lines_c4_r2l.txt 2>&1
python tools/ncu_kernels.py $OUT/raw_c4_r2l.csv > $OUT/ncu_kernels_c4_r2l.json 2>&1
python tools/ncu_traffic.py $OUT/raw_c4_r2l.csv c4 $OUT/ncu_c4_traffic.json
timeout 1200 python bench.py > $OUT/bench_r2l.json 2> $OUT/bench_r2l.err; echo "bench=$?"
python - <<PY
import json
d=json.load(open("$OUT/bench_r2l.json"))
print("C2", d["value"], d["ms_per_step"], "cold", d["cold"]["value"], "cpu", d["cpu_baseline"]["value"], "chain", d["roofline_chain"]["frac"])
s=d["secondary_c4"]; print("C4", s["value"], s["ms_per_step"], "cold", s["cold"]["value"], s["cold"]["ms_per_step"], "launches", s["gpu_launches"])
s=d["secondary_c3"]; print("C3", s["value"], s["ms_per_step"], "cold", s["cold"]["value"], "cpu", s["cpu_baseline"]["value"])
print("c5", d["c5_live"]["stream_copy_gbs"])
PY
bash tools/gpu_multirank.sh
bash tools/gpu_sanitize.sh r2l
