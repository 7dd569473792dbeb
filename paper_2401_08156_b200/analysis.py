"""Timeline and convergence analysis of replay outputs:
per-iteration S-state histograms from the assignment records, "stable after
k iterations" ("after a few iterations, GMLake will no
longer execute S2, S3, and S4"; fig:trace, L776-790), per-iteration peaks of
the (active, reserved) timeline, and policy grids over the fragmentation
limit and the sPool caps ("hyper-parameters ... empirically configured",
L625) for gml_replay to evaluate in one batch. Host-side arithmetic on the
records the GPU produced; the replay itself runs in K1."""
from __future__ import annotations

import numpy as np

STATES = ["S1", "S2", "S3", "S4", "S5", "bfc_hit", "bfc_new_segment"]


def record_states(records: np.ndarray) -> np.ndarray:
    """State field of assignment records (gml.h): 1..7, 0 for frees."""
    return ((np.asarray(records, dtype=np.uint64) >> np.uint64(34)) & np.uint64(7)).astype(np.int64)


def state_histograms(records: np.ndarray, iter_starts) -> np.ndarray:
    """[n_iterations, 7] counts of S1..S5, BFC hit, BFC new segment per
    iteration; iter_starts = event index of each iteration's first event
    (tracegen's side array; a final n may be included)."""
    st = record_states(records)
    bounds = list(iter_starts)
    if not bounds or bounds[-1] != len(st):
        bounds = bounds + [len(st)]
    out = np.zeros((len(bounds) - 1, 7), dtype=np.int64)
    for i in range(len(bounds) - 1):
        s = st[bounds[i]:bounds[i + 1]]
        s = s[s > 0]
        out[i] = np.bincount(s - 1, minlength=7)[:7]
    return out


def stable_after(hist: np.ndarray) -> int | None:
    """First iteration k from which no iteration executes S2, S3, S4 or S5
    (only S1 and the small path remain); None if the last iteration still
    does."""
    bad = hist[:, 1:5].sum(axis=1) > 0
    if bad[-1]:
        return None
    idx = np.nonzero(bad)[0]
    return 0 if len(idx) == 0 else int(idx[-1]) + 1


def iteration_peaks(timeline: np.ndarray, iter_starts) -> np.ndarray:
    """[n_iterations, 2] max (active, reserved) bytes per iteration from a
    [n_events, 2] timeline."""
    tl = np.asarray(timeline, dtype=np.uint64).reshape(-1, 2)
    bounds = list(iter_starts)
    if not bounds or bounds[-1] != len(tl):
        bounds = bounds + [len(tl)]
    return np.array([tl[bounds[i]:bounds[i + 1]].max(axis=0) for i in range(len(bounds) - 1)], dtype=np.uint64)


def policy_grid(capacity: int, limits_mib, spool_caps, flags: int = 0, byte_cap: int | None = None) -> list[dict]:
    """GMLake policies over frag_limit x spool_max_entries (one gml_replay
    evaluates the whole grid: every (trace, policy) is its own warp)."""
    MiB = 1 << 20
    return [{"kind": 2, "flags": flags, "capacity_bytes": capacity, "chunk_bytes": 2 * MiB,
             "small_threshold_bytes": 2 * MiB, "frag_limit_bytes": lim * MiB, "spool_max_entries": cap,
             "_pad": 0, "spool_max_inactive_bytes": capacity if byte_cap is None else byte_cap}
            for lim in limits_mib for cap in spool_caps]


def mem_reduction_ratio(reserved, gmlake_reserved) -> float:
    """MemReductionRatio = (sum Reserved - sum GMLakeReserved) / sum Reserved
    over matched workloads; Reserved = the baseline's
    (PyTorch, V0) peak reserved bytes."""
    if len(reserved) != len(gmlake_reserved) or not len(reserved):
        raise ValueError("workload lists must be non-empty and matched")
    a, b = float(sum(reserved)), float(sum(gmlake_reserved))
    if a == 0:
        raise ValueError("zero denominator")
    return (a - b) / a


def policy_report(stats_per_trace, names=None, base: int = 0) -> dict:
    """Per policy over a batch of traces: utilization =
    sum of peak active / sum of peak reserved, fragmentation = 1 - that,
    utilization from requested bytes (rounding padding NOT counted as used),
    mean padding, mean peak reserved, OOM traces, and MemReductionRatio vs
    policy `base` (V0 = PyTorch's caching allocator) over the traces both
    completed. stats_per_trace: [trace][policy] stats dicts."""
    GiB = float(1 << 30)
    n_pol = len(stats_per_trace[0])
    out = {}
    for p in range(n_pol):
        ss = [t[p] for t in stats_per_trace]
        a_ = sum(x["peak_active_bytes"] for x in ss)
        q_ = sum(x["peak_requested_bytes"] for x in ss)
        r_ = sum(x["peak_reserved_bytes"] for x in ss)
        ok = [i for i, t in enumerate(stats_per_trace) if t[p]["status"] == 0 and t[base]["status"] == 0]
        mrr = None
        if ok:
            mrr = mem_reduction_ratio([stats_per_trace[i][base]["peak_reserved_bytes"] for i in ok],
                                      [stats_per_trace[i][p]["peak_reserved_bytes"] for i in ok])
        key = names[p] if names else f"V{p}"
        out[key] = {"utilization": a_ / r_ if r_ else 1.0,
                    "fragmentation_pct": 100 * (1 - a_ / r_) if r_ else 0.0,
                    "utilization_requested": q_ / r_ if r_ else 1.0,
                    "padding_gib": (a_ - q_) / len(ss) / GiB,
                    "peak_reserved_gib": r_ / len(ss) / GiB,
                    "oom_traces": sum(x["status"] == 2 for x in ss),
                    "mem_reduction_vs_V%d" % base: mrr, "matched_traces": len(ok)}
    return out
