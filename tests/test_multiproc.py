"""N>1 host path on CPU: LPT sharding and the single stats all_gather, with
world_size 2 over gloo. Sharding must not change any
per-trace output: the oracle replays of the union of the shards equal the
replays of the whole batch."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2401_08156_b200.shard import gather_stats, lpt_shard


def test_lpt_properties():
    lengths = [5, 9, 1, 7, 7, 3, 2, 8]
    s = lpt_shard(lengths, 3)
    assert sorted(i for x in s for i in x) == list(range(8))
    loads = [sum(lengths[i] for i in x) for x in s]
    assert max(loads) - min(loads) <= max(lengths)
    assert lpt_shard(lengths, 1) == [list(range(8))]
    assert lpt_shard(lengths, 3) == s                      # deterministic
    assert lpt_shard([], 2) == [[], []]
    with pytest.raises(ValueError):
        lpt_shard(lengths, 0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.join(os.path.dirname(__file__)))
        import oracle_lib as O
        from tracegen import synth, policies as P
        traces = [synth.random_trace(100 + i, 200 + 37 * i, 10, size_lo=1, size_hi=64 << 20) for i in range(5)]
        pols = P.variants(capacity=1 << 30)[:4]
        mine = lpt_shard([len(t) for t in traces], world)[rank]
        recs = []
        for t in mine:
            for pol in pols:
                _, st = O.replay(traces[t], pol)
                recs.append(np.frombuffer(O.stats_bytes(st), dtype=np.uint8))
        local = torch.from_numpy(np.concatenate(recs) if recs else np.zeros(0, np.uint8))
        parts = gather_stats(local, len(mine) * len(pols))
        # the single-collective form (counts known from the deterministic shard)
        counts = [len(x) * len(pols) for x in lpt_shard([len(t) for t in traces], world)]
        parts1 = gather_stats(local, len(mine) * len(pols), counts=counts)
        assert all(torch.equal(a, b) for a, b in zip(parts, parts1))
        # gather_all: the same single collective, reassembled in global trace order
        from paper_2401_08156_b200.shard import gather_all, shard_plan
        plan = shard_plan([len(t) for t in traces], world, rank)
        assert plan.mine == mine
        full = gather_all(plan, local, len(pols))
        for t, tr in enumerate(traces):
            for p, pol in enumerate(pols):
                _, st = O.replay(tr, pol)
                assert full[t, p].tobytes() == O.stats_bytes(st), (t, p)
        if rank == 0:
            q.put(([p.numpy().tobytes() for p in parts], lpt_shard([len(t) for t in traces], world)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_matches_single_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts, shards = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # reassemble per trace and compare with a single-rank replay of everything
    import oracle_lib as O
    from tracegen import synth, policies as P
    traces = [synth.random_trace(100 + i, 200 + 37 * i, 10, size_lo=1, size_hi=64 << 20) for i in range(5)]
    pols = P.variants(capacity=1 << 30)[:4]
    got = {}
    for r, blob in enumerate(parts):
        arr = np.frombuffer(blob, dtype=np.uint8).reshape(-1, 272)
        for k, t in enumerate(shards[r]):
            for p in range(len(pols)):
                got[(t, p)] = arr[k * len(pols) + p].tobytes()
    assert len(got) == len(traces) * len(pols)
    for t, tr in enumerate(traces):
        for p, pol in enumerate(pols):
            _, st = O.replay(tr, pol)
            assert got[(t, p)] == O.stats_bytes(st), (t, p)
