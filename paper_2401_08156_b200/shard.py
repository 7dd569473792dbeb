"""Trace-parallel sharding across ranks.

Traces and policies are independent units, so ranks replay disjoint traces
with no data-path collective; the only exchange is one all_gather of the
per-(trace, policy) stats records after the replay. Host-side logic and
marshalling only: every replay runs in K1 through `gml_replay`.

    plan = shard_plan(lengths, world, rank)          # LPT by event count
    res = replay_sharded(lengths, get_trace, policies)
    res.stats[t][p]                                  # every trace, every rank
    res.assignments                                  # this rank's records
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass, field

import numpy as np


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


@dataclass
class ShardPlan:
    """Which global traces each rank replays (LPT)."""
    world: int
    rank: int
    n_traces: int
    shards: list = field(default_factory=list)     # per rank: ascending global trace indices

    @property
    def mine(self) -> list[int]:
        return self.shards[self.rank]

    def counts(self, n_policies: int) -> list[int]:
        """stats records per rank (every rank computes the same plan, so the
        gather needs no count exchange)."""
        return [len(s) * n_policies for s in self.shards]


def shard_plan(lengths, world: int, rank: int) -> ShardPlan:
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return ShardPlan(world, rank, len(lengths), lpt_shard(lengths, world))


def _dist_world(group=None):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def gather_stats(stats, n_local_units: int, group=None, counts=None):
    """All-gather the raw stats records (uint8 tensors of n_local_units * 272
    bytes) -> list of per-rank tensors. With `counts` (every rank's unit
    count, known when the shards are computed deterministically) this is the
    single collective of SURVEY §8(e); without, one more all_gather of the
    counts precedes it (ranks may hold different counts). Over gloo (CPU
    tests, shared-GPU exercises) device tensors are staged through the host,
    since gloo gathers host tensors only."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = stats.device
    if dev.type == "cuda" and dist.get_backend(group) == "gloo":
        dev = torch.device("cpu")
        stats = stats.cpu()
    if counts is None:
        n = torch.tensor([n_local_units], dtype=torch.int64, device=dev)
        ns = [torch.zeros_like(n) for _ in range(world)]
        dist.all_gather(ns, n, group=group)
        counts = [int(x.item()) for x in ns]
    mx = max(max(counts) * 272, 272)
    buf = torch.zeros(mx, dtype=torch.uint8, device=dev)
    buf[: stats.numel()] = stats.reshape(-1)[: n_local_units * 272]
    bufs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(bufs, buf, group=group)
    return [b[: c * 272] for b, c in zip(bufs, counts)]


def gather_all(plan: ShardPlan, local_stats, n_policies: int, group=None) -> np.ndarray:
    """One all_gather of every rank's stats records, reassembled in global
    trace order -> structured array [n_traces, n_policies] of gml_stats_t."""
    from . import gml
    out = np.zeros((plan.n_traces, n_policies), dtype=gml.STATS_DTYPE)
    if plan.world == 1:
        parts = [local_stats]
    else:
        parts = gather_stats(local_stats, len(plan.mine) * n_policies, group=group,
                             counts=plan.counts(n_policies))
    for r, part in enumerate(parts):
        if not plan.shards[r]:
            continue
        arr = gml.stats_from_bytes(part.cpu().numpy()).reshape(len(plan.shards[r]), n_policies)
        out[plan.shards[r]] = arr
    return out


@dataclass
class ShardedReplay:
    plan: ShardPlan
    batch: object                  # replay.DeviceBatch of this rank's traces (None if it has none)
    assignments: object            # int64 tensor [P, local events] or None
    local_stats: object            # uint8 tensor [len(mine) * P * 272]
    stats: np.ndarray              # gml_stats_t [n_traces, P], every rank's traces

    def stats_dicts(self) -> list[list[dict]]:
        from . import gml
        return [[gml.stats_dict(s) for s in row] for row in self.stats]

    def local_records(self, t: int):
        """this rank's assignment records of global trace t -> int64 tensor [P, len]"""
        k = self.plan.mine.index(t)
        off = self.batch.offsets.cpu().numpy()
        return self.assignments[:, int(off[k]):int(off[k + 1])]


def replay_sharded(lengths, get_trace, policies, group=None, device=None, stream=None,
                   with_assignments: bool = True, caps=None) -> ShardedReplay:
    """Replay a global batch of traces over the ranks of `group`: LPT shard
    by event count (`lengths`), each rank loads only its own traces
    (`get_trace(i)` -> packed u64 events) and replays them x `policies`
    with K1 (gml_replay) on `device`, then ONE all_gather of the stats.
    Assignment records stay rank-local. Without an initialised process
    group this is a single-rank replay of the whole batch."""
    import torch
    from . import replay as R
    world, rank = _dist_world(group)
    plan = shard_plan(lengths, world, rank)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    V = len(policies)
    batch, asg = None, None
    if plan.mine:
        traces = [np.asarray(get_trace(i), dtype=np.uint64) for i in plan.mine]
        for i, tr in zip(plan.mine, traces):
            if len(tr) != int(lengths[i]):
                raise ValueError(f"trace {i}: {len(tr)} events, plan says {int(lengths[i])}")
        ctx = torch.cuda.device(dev)
        with ctx:
            batch = R.upload(traces, dev)
            asg, st = R.run(batch, policies, with_assignments=with_assignments, stream=stream, caps=caps)
            (stream or torch.cuda.current_stream(dev)).synchronize()
    else:
        st = torch.zeros(0, dtype=torch.uint8, device=dev)
    stats = gather_all(plan, st, V, group=group)
    return ShardedReplay(plan, batch, asg, st, stats)
