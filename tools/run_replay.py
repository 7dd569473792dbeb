"""Run gml_replay on a bench workload a few times (for ncu / per-unit cycle
debugging). Not part of the timed bench."""
import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--policies", default="")
    ap.add_argument("--caps", default="tight", help="tight (the classes of a first replay) | cold (no hint each rep) | P,S,IV,B (fixed hint)")
    args = ap.parse_args()
    import torch
    import bench
    from paper_2401_08156_b200 import replay as R, gml
    W = bench.Workload(args.workload, 1)
    traces, pols, desc = W.load(list(range(W.n))), W.pols, W.desc
    if args.policies:
        pols = [pols[int(i)] for i in args.policies.split(",")]
    batch = R.upload(traces, "cuda:0")
    caps = np.zeros((len(traces) * len(pols), 4), dtype=np.uint32)
    asg, st = R.run(batch, pols, caps=caps)
    stats = R.decode_stats(st, len(traces), len(pols))
    # caps now hold the classes this replay ended in (written back by gml_replay)
    if args.caps not in ("tight", "cold"):
        caps[:] = np.array([int(x) for x in args.caps.split(",")], dtype=np.uint32)
    R.run(batch, pols, caps=caps, assignments=asg, stats=st)   # settle caps
    hint = caps.copy()
    for _ in range(args.reps):
        caps[:] = 0 if args.caps == "cold" else hint
        torch.cuda.synchronize()
        t = time.perf_counter()
        torch.cuda.nvtx.range_push("timed")
        R.run(batch, pols, caps=caps, assignments=asg, stats=st)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
        print(f"{desc}: {1e3*(time.perf_counter()-t):.2f} ms wall, kernel {gml.gml_last_kernel_ms():.2f} ms",
              file=sys.stderr)


if __name__ == "__main__":
    main()
