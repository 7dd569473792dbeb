"""DEBUG PROBE (not product code): C4 step time (device events around the
gml_replay call, as bench.py times it) vs the kernels' own time, with and
without the nvidia-smi clock sampler running. Usage (GPU): python tools/c4_hostgap.py"""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("GML_C4_PER_GPU", "512")

import numpy as np  # noqa: E402


def main():
    import torch
    import bench
    from paper_2401_08156_b200 import replay as R, gml
    W = bench.Workload("c4", 1)
    tr = W.load(list(range(W.n)))
    st = torch.cuda.Stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    with torch.cuda.stream(st):
        b = R.upload(tr, "cuda:0")
        asg = torch.empty((8, b.total), dtype=torch.int64, device="cuda")
        sts = torch.empty((len(tr) * 8 * 272,), dtype=torch.uint8, device="cuda")
    st.synchronize()
    caps = np.zeros((len(tr) * 8, 4), dtype=np.uint32)
    for _ in range(3):
        R.run(b, W.pols, stream=st, caps=caps, assignments=asg, stats=sts)
    hint = caps.copy()

    def steps(k, cold):
        ea = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        eb = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        kern, wall = [], []
        torch.cuda.synchronize()
        for i in range(k):
            caps[:] = 0 if cold else hint
            with torch.cuda.stream(st):
                flush.zero_()
            ea[i].record(st)
            t = time.perf_counter()
            R.run(b, W.pols, stream=st, caps=caps, assignments=asg, stats=sts)
            wall.append(1e3 * (time.perf_counter() - t))
            eb[i].record(st)
            kern.append(gml.gml_last_kernel_ms())
        torch.cuda.synchronize()
        dev = [a.elapsed_time(c) for a, c in zip(ea, eb)]
        print("  per step device:", " ".join(f"{x:.1f}" for x in dev), " wall:", " ".join(f"{x:.1f}" for x in wall), flush=True)
        return np.mean(dev), np.mean(kern), np.mean(wall)

    for label in ("hinted", "cold", "hinted+smi", "cold+smi"):
        cold = label.startswith("cold")
        if "smi" in label:
            with bench.Clocks(0):
                d, k, w = steps(5, cold)
        else:
            d, k, w = steps(5, cold)
        print(f"{label:12s} device {d:7.2f} ms  kernels {k:7.2f} ms  host wall {w:7.2f} ms", flush=True)


if __name__ == "__main__":
    main()
