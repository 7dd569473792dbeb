"""DEBUG PROBE (not product code): how long would each C2 GMLake unit take if
its small-path (BFC) events and its VMM-path events ran on two warps? Replays,
per policy, the sub-trace of VMM-path events alone and of small-path events
alone (decisions are the same as in the full trace while capacity never
binds) with per-unit cycle counters (GML_UNIT_CYCLES=1).
Usage (GPU): GML_UNIT_CYCLES=1 python tools/split_probe.py [c2|c3]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402


def split(ev, thr):
    ev = np.asarray(ev, dtype=np.uint64)
    is_free = (ev >> np.uint64(63)).astype(bool)
    slot = ((ev >> np.uint64(40)) & np.uint64(0x7FFFFF)).astype(np.int64)
    raw = (ev & np.uint64((1 << 40) - 1)).astype(np.int64)
    big = np.zeros(len(ev), dtype=bool)
    last = {}
    for i in range(len(ev)):
        s = slot[i]
        if is_free[i]:
            big[i] = last.pop(s)
        else:
            big[i] = raw[i] >= thr
            last[s] = big[i]
    return ev[big], ev[~big]


def main():
    import torch  # noqa: F401
    import bench
    from paper_2401_08156_b200 import replay as R, gml
    wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
    W = bench.Workload(wl, 1)
    tr = W.load([0])[0]
    pols = W.pols
    for v, p in enumerate(pols):
        if p["kind"] != 2:
            continue
        thr = max(p.get("small_threshold_bytes", 2 << 20), p["frag_limit_bytes"] if p.get("flags", 0) & 16 else 0)
        vm, sm = split(tr, thr)
        for name, t in (("full", np.asarray(tr, dtype=np.uint64)), ("vmm", vm), ("small", sm)):
            b = R.upload([t], "cuda:0")
            caps = np.zeros((1, 4), dtype=np.uint32)
            R.run(b, [p], caps=caps)
            R.run(b, [p], caps=caps)
            print(f"V{v} {name} events {len(t)} kernel {gml.gml_last_kernel_ms():.2f} ms", flush=True)


if __name__ == "__main__":
    main()
