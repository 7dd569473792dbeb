"""Small replays for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck) of K0 + K1: fig:intro, fuzz traces with tight capacities (OOM
paths), a ragged batch with empty traces, an irregular trace and a C2
prefix, all 8 policies plus flag variants; shared-memory arenas by default,
global-memory arenas with GML_FORCE_GLOBAL=1, the throughput placement (path
units) with GML_SAN_THROUGHPUT=1. Results are checked against
the oracle so a sanitizer run is also a parity run."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402

MiB = 1 << 20
GiB = 1 << 30


def main():
    import torch
    import oracle_lib as O
    from paper_2401_08156_b200 import replay as R
    from tracegen import synth
    from tracegen import policies as P
    traces = [synth.fig_intro(), np.zeros(0, np.uint64)]
    traces += [synth.random_trace(s, 250, 12, sizes=[1, 511, 513, 300 * 1024, 1536 * 1024, 2 * MiB,
                                                     3 * MiB, 6 * MiB, 14 * MiB, 40 * MiB]) for s in range(6)]
    traces += [synth.lognormal_trace(3, 2, 30, 50e6, extra_frac=0.3, interleave_frac=0.3, small_frac=0.2),
               synth.config_c2(iters=2)[0][:6000]]
    import os
    if os.environ.get("GML_SAN_THROUGHPUT"):
        # > 4 units per SM: the throughput placement (path units, ledger, merge)
        traces = traces * 8
    n_bad = 0
    for cap in (48 * MiB, 80 * GiB):
        pols = P.variants(capacity=cap)
        for p in pols[2:]:
            p["frag_limit_bytes"] = 2 * MiB if cap < GiB else p["frag_limit_bytes"]
        pols[7]["spool_max_entries"] = 3
        pols.append(P.policy(P.GMLAKE, P.F_S1_PBLOCK_FIRST | P.F_NO_COMPANION, capacity=cap,
                             frag_limit=4 * MiB, spool_max_inactive_bytes=16 * MiB))
        batch = R.upload(traces)
        asg, st = R.run(batch, pols)
        torch.cuda.synchronize()
        stats = R.decode_stats(st, len(traces), len(pols))
        a = asg.cpu().numpy().view(np.uint64)
        off = 0
        for t, tr in enumerate(traces):
            for p, pol in enumerate(pols):
                ao, so = O.replay(tr, pol)
                if stats[t][p] != so or not np.array_equal(a[p, off:off + len(tr)], ao):
                    n_bad += 1
            off += len(tr)
    print(f"sanitize_replay: {len(traces)} traces, parity mismatches: {n_bad}")
    sys.exit(1 if n_bad else 0)


if __name__ == "__main__":
    main()
