"""f4: timeline + convergence on the GPU (fig:trace analogue, PAPER.md
L766-791) and a policy grid over the fragmentation limit x sPool cap
(L563-572, L625), each evaluated in one gml_replay batch.

    python tools/convergence.py > profiles/<round>/convergence.json
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402

GiB = 1 << 30


def main():
    import torch
    import __graft_entry__ as ge
    ge.build()
    from paper_2401_08156_b200 import analysis as An, gml, replay as R
    from tracegen import policies as P, synth
    out = {"workloads": {}, "grid": {}}
    work = {"C2": [synth.config_c2()], "C3": [synth.config_c3(r) for r in range(8)]}
    for name, items in work.items():
        traces = [ev for ev, _ in items]
        pols = P.variants(capacity=80 * GiB)
        batch = R.upload(traces)
        tl = torch.zeros((len(pols), batch.total, 2), dtype=torch.int64, device="cuda")
        asg, st = R.run(batch, pols, timeline=tl)
        torch.cuda.synchronize()
        a = asg.cpu().numpy().view(np.uint64)
        t = tl.cpu().numpy().view(np.uint64)
        stats = R.decode_stats(st, len(traces), len(pols))
        res = []
        off = 0
        for ti, (ev, starts) in enumerate(items):
            n = len(ev)
            for p in range(len(pols)):
                h = An.state_histograms(a[p, off:off + n], starts)
                pk = An.iteration_peaks(t[p, off:off + n], starts)
                s = stats[ti][p]
                res.append({"trace": ti, "policy": f"V{p}", "stable_after": An.stable_after(h),
                            "iter_S_counts_first4": h[:4, :5].tolist(), "iter_S_counts_last": h[-1, :5].tolist(),
                            "iter_peak_active_gib": (pk[:, 0] / GiB).round(3).tolist(),
                            "iter_peak_reserved_gib": (pk[:, 1] / GiB).round(3).tolist(),
                            "utilization": s["peak_active_bytes"] / max(s["peak_reserved_bytes"], 1)})
            off += n
        out["workloads"][name] = res
        # grid: frag limit x sPool count cap
        limits, caps = [2, 4, 8, 16, 32, 64, 128, 256, 512], [16, 64, 512, 4096]
        grid = An.policy_grid(80 * GiB, limits, caps)
        t0 = time.perf_counter()
        _, gst = R.run(batch, grid, with_assignments=False)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        gs = R.decode_stats(gst, len(traces), len(grid))
        cells = []
        for gi, pol in enumerate(grid):
            act = sum(gs[ti][gi]["peak_active_bytes"] for ti in range(len(traces)))
            rsv = sum(gs[ti][gi]["peak_reserved_bytes"] for ti in range(len(traces)))
            cells.append({"frag_limit_mib": pol["frag_limit_bytes"] >> 20, "spool_max_entries": pol["spool_max_entries"],
                          "utilization": act / max(rsv, 1), "peak_reserved_gib_mean": rsv / len(traces) / GiB,
                          "n_evict": sum(gs[ti][gi]["n_evict"] for ti in range(len(traces)))})
        out["grid"][name] = {"units": len(traces) * len(grid), "wall_s": dt,
                             "event_replays": int(batch.total * len(grid)), "cells": cells}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
