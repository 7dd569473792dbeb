set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_r2h.log 2>&1; echo build=$?
for pol in 3 4; do
  timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:k_replay -c 2 \
     -o /tmp/prof_v$pol python tools/run_replay.py --workload c2 --reps 1 --policies $pol > $OUT/ncu_v${pol}.log 2>&1; echo "ncu v$pol=$?"
  ncu -i /tmp/prof_v$pol.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_v$pol.csv 2>/dev/null
  python tools/ncu_lines.py /tmp/src_v$pol.csv 80 > $OUT/hot_lines_c2_v${pol}_r2h.txt 2>&1
  ncu -i /tmp/prof_v$pol.ncu-rep --page raw --csv > $OUT/raw_c2_v${pol}_r2h.csv 2>/dev/null
  head -c 300 $OUT/hot_lines_c2_v${pol}_r2h.txt; echo
done
timeout 900 python bench.py --no-c5 > $OUT/bench_r2h.json 2> $OUT/bench_r2h.err; echo "bench=$?"
python - <<PY
import json
d=json.load(open("$OUT/bench_r2h.json"))
print("C2", d["value"], d["ms_per_step"], "cold", d["cold"]["value"])
s=d["secondary_c4"]; print("C4", s["value"], s["ms_per_step"], "cold", s["cold"]["value"], s["cold"]["ms_per_step"], "launches", s["gpu_launches"])
PY
