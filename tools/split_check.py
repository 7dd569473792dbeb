"""DEBUG CHECK (not product code): replay a bench workload with split units
(default) and with GML_NO_SPLIT semantics (via the env var in a subprocess is
not needed: the library reads it per call) and compare records + stats; print
kernel times. Usage (GPU): python tools/split_check.py [c2|c3] [reps]"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402


def main():
    import torch
    import bench
    from paper_2401_08156_b200 import replay as R, gml
    wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    W = bench.Workload(wl, 1)
    traces, pols = W.load(list(range(W.n))), W.pols
    batch = R.upload(traces, "cuda:0")
    out = {}
    for mode in ("serial", "split"):
        if mode == "serial":
            os.environ["GML_NO_SPLIT"] = "1"
        else:
            os.environ.pop("GML_NO_SPLIT", None)
        caps = np.zeros((len(traces) * len(pols), 4), dtype=np.uint32)
        asg, st = R.run(batch, pols, caps=caps)
        ts = []
        for _ in range(reps):
            R.run(batch, pols, caps=caps, assignments=asg, stats=st)
            torch.cuda.synchronize()
            ts.append(gml.gml_last_kernel_ms())
        out[mode] = (asg.cpu().numpy().copy(), st.cpu().numpy().copy())
        print(f"{wl} {mode}: kernel ms {' '.join(f'{t:.2f}' for t in ts)} launches {gml.gml_last_launch_count()}", flush=True)
    a0, s0 = out["serial"]
    a1, s1 = out["split"]
    print("records equal:", np.array_equal(a0, a1), "stats equal:", np.array_equal(s0, s1))
    if not np.array_equal(s0, s1):
        import torch
        d0 = R.decode_stats(torch.from_numpy(s0), len(traces), len(pols))
        d1 = R.decode_stats(torch.from_numpy(s1), len(traces), len(pols))
        for t in range(len(traces)):
            for p in range(len(pols)):
                x, y = d0[t][p], d1[t][p]
                for k in x:
                    if x[k] != y[k]:
                        print("trace", t, "policy", p, k, x[k], y[k])
    if not np.array_equal(a0, a1):
        bad = np.argwhere(a0 != a1)
        print("first record diffs:", bad[:10].tolist())


if __name__ == "__main__":
    main()
