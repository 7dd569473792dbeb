"""Aggregate an `ncu --page source --csv --print-source cuda,sass` export by
CUDA source line: warp-stall samples and executed instructions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur, agg, src = None, {}, {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] == "Line No":
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    if r[1]:
        src[(cur, ln)] = r[1]
    try:
        s, ex = int(r[4] or 0), int(r[7] or 0)
    except ValueError:
        continue
    a = agg.setdefault((cur, ln), [0, 0])
    a[0] += s
    a[1] += ex
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total stall samples {ts}, executed warp instructions {ti}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0]:8d} {100 * v[0] / ts:5.1f}%  inst {v[1]:11d} {100 * v[1] / ti:5.1f}%  {k[0]}:{k[1]}  {src.get(k, '')[:100]}")
print()
print("by executed instructions:")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{v[0]:8d} {100 * v[0] / ts:5.1f}%  inst {v[1]:11d} {100 * v[1] / ti:5.1f}%  {k[0]}:{k[1]}  {src.get(k, '')[:100]}")
