"""Request-size histogram of the bench configurations against the small-path
threshold (2 MiB) and the fragmentation limit (128 MiB,
PAPER.md L572): how many mallocs and bytes each reading of the limit (D8:
filters candidate blocks; D8': gates requests) sends down which path.
Writes profiles/size_histogram.json and prints a markdown table."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

MiB = 1 << 20
EDGES = [0, 2 * MiB, 32 * MiB, 128 * MiB, 512 * MiB, 1 << 62]
NAMES = ["< 2 MiB", "2-32 MiB", "32-128 MiB", "128-512 MiB", ">= 512 MiB"]


def hist(ev):
    m = ev[(ev >> np.uint64(63)) == 0] & np.uint64((1 << 40) - 1)
    m = m.astype(np.float64)
    out = []
    for lo, hi, nm in zip(EDGES[:-1], EDGES[1:], NAMES):
        sel = (m >= lo) & (m < hi)
        out.append({"bin": nm, "mallocs": int(sel.sum()), "malloc_frac": float(sel.mean()),
                    "bytes_frac": float(m[sel].sum() / m.sum())})
    return {"mallocs": int(len(m)), "distinct_sizes": int(len(np.unique(m))), "bins": out}


def main():
    from tracegen import synth
    res = {"C2": hist(synth.config_c2()[0]),
           "C3 (rank 0)": hist(synth.config_c3(0)[0]),
           "C4 (every 64th of 4096)": hist(np.concatenate([synth.config_c4(i)[0] for i in range(0, 4096, 64)]))}
    (ROOT / "profiles" / "size_histogram.json").write_text(json.dumps(res, indent=1))
    print("| config | mallocs | distinct sizes | " + " | ".join(NAMES) + " |")
    print("|---|---|---|" + "---|" * len(NAMES))
    for k, v in res.items():
        cells = [f"{b['malloc_frac']*100:.1f} % ({b['bytes_frac']*100:.1f} % of bytes)" for b in v["bins"]]
        print(f"| {k} | {v['mallocs']} | {v['distinct_sizes']} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main()
