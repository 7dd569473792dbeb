#!/bin/bash
# Round-3 GPU session: bench, launch list, ncu full captures (every kernel of
# one gml_replay), the C2 chain profile. Usage (under gpurun): bash tools/gpu_round3.sh <tag>
set -u
TAG=${1:-r3}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1; echo "build=$?"
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench=$?"; head -c 600 $OUT/bench_$TAG.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/bench_ncu_$TAG.log 2>&1; echo "ncu_launches=$?"
prof() {  # name, workload [extra ncu args]
  local name=$1; local wl=$2; shift 2
  timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" "$@" \
      -k regex:"k_replay|k_ledger|k_merge|k_max_slot" -c 16 -o /tmp/prof_$name python tools/run_replay.py --workload $wl --reps 1 > $OUT/ncu_full_$name.log 2>&1; echo "ncu_full_$name=$?"
  ncu -i /tmp/prof_$name.ncu-rep --page raw --csv > $OUT/raw_$name.csv 2>/dev/null
  ncu -i /tmp/prof_$name.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_$name.csv 2>/dev/null
  python tools/ncu_lines.py /tmp/src_$name.csv 60 > $OUT/hot_lines_$name.txt 2>&1
  python tools/ncu_kernels.py $OUT/raw_$name.csv > $OUT/ncu_kernels_$name.json 2>&1
  python tools/ncu_traffic.py $OUT/raw_$name.csv $wl $OUT/ncu_${wl}_traffic.json
}
prof c2_$TAG c2
GML_C4_PER_GPU=512 prof c4_$TAG c4 --replay-mode application
bash tools/gpu_units.sh $TAG > $OUT/units_$TAG.log 2>&1; echo "units=$?"
du -sh $OUT
