"""Per-kernel summary of an `ncu --page raw --csv` export (key metrics)."""
import csv
import json
import sys

KEYS = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "lts__t_bytes.sum", "l1tex__t_sector_hit_rate.pct",
        "launch__shared_mem_per_block_dynamic", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
rows = list(csv.reader(open(sys.argv[1])))
hdr, units, data = rows[0], rows[1], rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
out = []
for d in data:
    out.append({k: (d[idx[k]].strip() + " " + units[idx[k]]).strip() for k in KEYS if k in idx})
print(json.dumps(out, indent=1))
