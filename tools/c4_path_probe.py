"""DEBUG PROBE (not product code): would C4 (throughput placement) gain from
replaying each GMLake unit's VMM path and small path as separate units (the
small path in the high-occupancy BFC family)? Times, on the C4 batch:
full traces x GMLake policies, full x BFC policies, VMM-only sub-traces x
GMLake policies, small-only sub-traces x BFC-torch (standing in for the
GMLake small paths). Usage (GPU): python tools/c4_path_probe.py [n_traces]"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

import numpy as np  # noqa: E402


def main():
    import torch
    import bench
    from split_probe import split
    from paper_2401_08156_b200 import replay as R, gml
    from concurrent.futures import ProcessPoolExecutor
    per = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    os.environ["GML_C4_PER_GPU"] = str(per)
    W = bench.Workload("c4", 1)
    traces = W.load(list(range(W.n)))
    pols = W.pols
    with ProcessPoolExecutor(16) as ex:
        s2 = list(ex.map(split, traces, [2 << 20] * len(traces), chunksize=8))
        s128 = list(ex.map(split, traces, [128 << 20] * len(traces), chunksize=8))

    def t(trs, ps, reps=3):
        b = R.upload(trs, "cuda:0")
        caps = np.zeros((len(trs) * len(ps), 4), dtype=np.uint32)
        asg, st = R.run(b, ps, caps=caps)
        R.run(b, ps, caps=caps, assignments=asg, stats=st)
        ms = []
        for _ in range(reps):
            R.run(b, ps, caps=caps, assignments=asg, stats=st)
            torch.cuda.synchronize()
            ms.append(gml.gml_last_kernel_ms())
        return min(ms)

    ev = sum(len(x) for x in traces)
    print(f"events {ev}, vmm(2M) {sum(len(a) for a, _ in s2)}, vmm(128M) {sum(len(a) for a, _ in s128)}", flush=True)
    print(f"full x 8 policies: {t(traces, pols):.1f} ms", flush=True)
    print(f"full x V2-V7: {t(traces, pols[2:]):.1f} ms", flush=True)
    print(f"full x V0,V1: {t(traces, pols[:2]):.1f} ms", flush=True)
    print(f"vmm2M x V3-V7: {t([a for a, _ in s2], pols[3:]):.1f} ms", flush=True)
    print(f"vmm128M x V2: {t([a for a, _ in s128], pols[2:3]):.1f} ms", flush=True)
    print(f"small2M x V0 x5 (as 5 copies): {t([b for _, b in s2] * 5, pols[:1]):.1f} ms", flush=True)
    print(f"small128M x V0: {t([b for _, b in s128], pols[:1]):.1f} ms", flush=True)
    # everything of the path scheme in one call is not expressible (cross product); a
    # combined BFC-family load: full x V0,V1 + small parts as V0
    bfc_all = list(traces) * 2 + [b for _, b in s2] * 5 + [b for _, b in s128]
    print(f"all BFC-family work as V0 units: {t(bfc_all, pols[:1]):.1f} ms", flush=True)


if __name__ == "__main__":
    main()
