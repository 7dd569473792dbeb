"""N>1 path on the GPU: two ranks (gloo, both on
cuda:0 -- this pool gives one GPU per call) LPT-shard a global batch, replay
their shards with K1 through gml_replay and gather the stats with ONE
all_gather (`shard.replay_sharded`). The gathered stats and every rank's
assignment records must equal the CPU oracle's and the N=1 replay's, byte
for byte: sharding never changes a per-trace output."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MiB = 1 << 20
GiB = 1 << 30


def _batch():
    from tracegen import synth
    from tracegen import policies as P
    traces = [synth.fig_intro()]
    traces += [synth.random_trace(300 + i, 300 + 53 * i, 16, size_lo=1, size_hi=96 * MiB) for i in range(4)]
    traces += [synth.lognormal_trace(7, 3, 40, 60e6, extra_frac=0.3, interleave_frac=0.3, small_frac=0.2),
               synth.config_c4(37, iters=2)[0]]
    pols = P.variants(capacity=8 * GiB)
    return traces, pols


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2401_08156_b200.shard import replay_sharded
        traces, pols = _batch()
        res = replay_sharded([len(t) for t in traces], lambda i: traces[i], pols, device="cuda:0")
        recs = {t: res.local_records(t).cpu().numpy().view(np.uint64).copy() for t in res.plan.mine}
        q.put((rank, res.plan.shards, res.stats.tobytes(), recs))
    finally:
        dist.destroy_process_group()


def test_two_ranks_replay_sharded_matches_oracle_and_single_rank():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge
    ge.build()
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    got.sort(key=lambda x: x[0])
    traces, pols = _batch()
    shards = got[0][1]
    assert got[1][1] == shards and sorted(shards[0] + shards[1]) == list(range(len(traces)))
    assert shards[0] and shards[1]                      # both ranks replay something
    assert got[0][2] == got[1][2]                        # every rank holds the same gathered stats

    import oracle_lib as O
    from paper_2401_08156_b200 import gml
    from paper_2401_08156_b200.shard import replay_sharded
    stats = np.frombuffer(got[0][2], dtype=gml.STATS_DTYPE).reshape(len(traces), len(pols))
    one = replay_sharded([len(t) for t in traces], lambda i: traces[i], pols, device="cuda:0")
    assert one.plan.world == 1 and one.stats.tobytes() == got[0][2]      # N=1 == N=2
    for rank, _, _, recs in got:
        for t, rec in recs.items():
            assert t in shards[rank]
            assert np.array_equal(rec, one.local_records(t).cpu().numpy().view(np.uint64))
            for p, pol in enumerate(pols):
                a_o, s_o = O.replay(traces[t], pol)
                assert np.array_equal(rec[p], a_o), (rank, t, p)
                assert gml.stats_dict(stats[t, p]) == s_o, (t, p)
