"""Trace-parallel sharding across ranks.

Traces and policies are independent units, so ranks replay disjoint traces
with no data-path collective; the only exchange is one all_gather of the
per-(trace, policy) stats records after the replay. Host-side logic only.
"""
from __future__ import annotations

import heapq


def lpt_shard(lengths, world: int) -> list[list[int]]:
    """Longest-processing-time assignment of trace indices to `world` ranks
    by event count. Deterministic: ties broken by lower index / lower rank.
    Each rank's list is returned in ascending trace order."""
    if world < 1:
        raise ValueError("world must be >= 1")
    heap = [(0, r) for r in range(world)]
    out: list[list[int]] = [[] for _ in range(world)]
    for i in sorted(range(len(lengths)), key=lambda i: (-int(lengths[i]), i)):
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + int(lengths[i]), r))
    return [sorted(x) for x in out]


def gather_stats(stats, n_local_units: int, group=None, counts=None):
    """All-gather the raw stats records (uint8 tensors of n_local_units * 272
    bytes) -> list of per-rank tensors. With `counts` (every rank's unit
    count, known when the shards are computed deterministically) this is the
    single collective of SURVEY §8(e); without, one more all_gather of the
    counts precedes it (ranks may hold different counts)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = stats.device
    if counts is None:
        n = torch.tensor([n_local_units], dtype=torch.int64, device=dev)
        ns = [torch.zeros_like(n) for _ in range(world)]
        dist.all_gather(ns, n, group=group)
        counts = [int(x.item()) for x in ns]
    mx = max(counts) * 272
    buf = torch.zeros(mx, dtype=torch.uint8, device=dev)
    buf[: stats.numel()] = stats
    bufs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf, group=group)
    return [b[: c * 272] for b, c in zip(bufs, counts)]
