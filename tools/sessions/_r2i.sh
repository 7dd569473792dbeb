set -u
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_r2i.log 2>&1; echo build=$?
python tools/build_variants.py "ev1=GML_EV_LOAD=1" "ev2=GML_EV_LOAD=2" >> $OUT/build_r2i.log 2>&1
cp paper_2401_08156_b200/libgml.so build/libgml_base.so
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool initcheck --error-exitcode 9 --print-limit 20 python tools/sanitize_replay.py > $OUT/sanitize_r2i_smem_initcheck.log 2>&1; echo "smem initcheck rc=$? $(grep -E 'SUMMARY' $OUT/sanitize_r2i_smem_initcheck.log)"
GML_FORCE_GLOBAL=1 timeout 1500 $CS --tool initcheck --error-exitcode 9 --print-limit 20 python tools/sanitize_replay.py > $OUT/sanitize_r2i_global_initcheck.log 2>&1; echo "global initcheck rc=$? $(grep -E 'SUMMARY' $OUT/sanitize_r2i_global_initcheck.log)"
for V in base ev1 ev2; do
  GML_LIB=build/libgml_$V.so GML_C4_PER_GPU=512 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --replay-mode application \
    --clock-control none --nvtx --nvtx-include "timed/" -k regex:k_replay --csv python tools/run_replay.py --workload c4 --reps 1 > $OUT/dram_c4_$V.csv 2>/dev/null
  python - $OUT/dram_c4_$V.csv $V <<'PY'
import csv, io, sys
txt = open(sys.argv[1]).read(); st = txt.find('"ID"')
tot = {}
for r in csv.DictReader(io.StringIO(txt[st:])):
    u = r["Metric Unit"]; v = float(r["Metric Value"].replace(",", ""))
    mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1, "msecond": 1, "us": 1e-3, "usecond": 1e-3, "ns": 1e-6, "nsecond": 1e-6}.get(u, 1)
    tot[r["Metric Name"]] = tot.get(r["Metric Name"], 0) + v * mul
print(sys.argv[2], {k: round(v / 1e9, 3) if "bytes" in k else round(v, 2) for k, v in tot.items()})
PY
done
for r in 1 2; do for V in base ev1 ev2; do
  GML_LIB=build/libgml_$V.so GML_C4_PER_GPU=512 timeout 600 python tools/run_replay.py --workload c4 --reps 2 2>&1 | tail -1 | sed "s|^|$V c4: |"
done; done
bash tools/gpu_units.sh r2i
