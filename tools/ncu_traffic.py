"""DRAM traffic per replay step from an `ncu --set full --page raw --csv`
export of the K1 launches of ONE gml_replay (tools/run_replay.py --reps 1):
writes profiles/ncu_<workload>_traffic.json, which bench.py reports as
roofline.traffic."""
import csv
import json
import sys

raw, workload, out = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tot, n, missing, inst, inst_missing = 0.0, 0, 0, 0.0, 0
for d in data:
    if not any(k in d[idx["Kernel Name"]] for k in ("k_replay", "k_ledger", "k_merge", "k_max_slot")):
        continue
    n += 1
    try:
        x = float(d[idx["smsp__inst_executed.sum"]].replace(",", ""))
    except (KeyError, ValueError):
        x = float("nan")
    if x == x:
        inst += x
    else:
        inst_missing += 1
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        v = d[idx[k]].replace(",", "").strip()
        try:
            x = float(v)
        except ValueError:
            x = float("nan")
        if x != x:                         # n/a or -nan: counter not collected for this launch
            missing += 1
            continue
        tot += x * scale.get(units[idx[k]].strip(), 1)
json.dump({"source": f"ncu --set full, tools/run_replay.py --workload {workload} --reps 1 ({n} launches of one gml_replay: K0, K1 / K1s / K1p, K1l, K1m)",
           "dram_bytes_per_launch": tot, "kernels_without_dram_counters": missing,
           "warp_instructions_per_launch": inst if not inst_missing else None,
           "kernels_without_instruction_counts": inst_missing,
           "note": "sum over every kernel launch of one replay step"
                   + (f"; {missing} counters of {2 * n} were not collected (ncu reported nan): a lower bound"
                      if missing else "")}, open(out, "w"), indent=1)
print(out, tot, n, missing)
