"""Split units (csrc/split_kernel.cuh): in the latency placement a GMLake unit
replays its VMM path and its small path on two warps of one CTA plus a
ledger warp. The split is exact only while neither path fails a capacity
check; every other outcome must be handed to the single-warp replay. These
tests check both sides: split results equal the oracle's and the single-warp
K1's, and each fallback cause (capacity sum, OOM, invalid trace, table
overflow) is re-run and still equals the oracle."""
import os

import numpy as np
import pytest

import oracle_lib as O
from tracegen import pack, synth
from tracegen import policies as P

pytestmark = pytest.mark.gpu

MiB = 1 << 20
GiB = 1 << 30


@pytest.fixture(scope="module")
def R():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge
    ge.build()
    from paper_2401_08156_b200 import replay
    return replay


def _run(R, traces, pols, caps=None, no_split=False):
    import torch
    from paper_2401_08156_b200 import gml
    if no_split:
        os.environ["GML_NO_SPLIT"] = "1"
    try:
        batch = R.upload(traces)
        sent = torch.full((len(pols), max(batch.total, 1)), -1, dtype=torch.int64, device="cuda")
        asg, st = R.run(batch, pols, caps=caps, assignments=sent)
        torch.cuda.synchronize()
        split = gml.gml_last_split_count()
    finally:
        os.environ.pop("GML_NO_SPLIT", None)
    return asg.cpu().numpy().view(np.uint64), R.decode_stats(st, len(traces), len(pols)), split


def _check_oracle(traces, pols, a, stats):
    off = 0
    for t, tr in enumerate(traces):
        for p, pol in enumerate(pols):
            ao, so = O.replay(tr, pol)
            assert stats[t][p] == so, (t, p, {k: (stats[t][p][k], so[k]) for k in so if stats[t][p][k] != so[k]})
            got = a[p, off:off + len(tr)]
            assert np.array_equal(got, ao), (t, p, int(np.nonzero(got != ao)[0][0]))
        off += len(tr)


def test_split_units_equal_single_warp_and_oracle(R):
    """C3 rank traces x V0-V7: the 6 GMLake units of each trace run split,
    none falls back, and records + stats equal the single-warp replay's and
    the oracle's."""
    traces = [synth.config_c3(r)[0] for r in (0, 5)]
    pols = P.variants(capacity=80 * GiB)
    a1, s1, (n_split, n_rerun) = _run(R, traces, pols)
    assert (n_split, n_rerun) == (12, 0)
    a0, s0, (m_split, _) = _run(R, traces, pols, no_split=True)
    assert m_split == 0
    assert np.array_equal(a0, a1) and s0 == s1
    _check_oracle(traces, pols, a1, s1)


def test_split_capacity_sum_falls_back(R):
    """Each path alone fits the capacity but their reserved bytes together do
    not: the split result would differ from the interleaved replay (the
    capacity checks see the other path's reserve), so the unit is re-run by
    the single-warp K1 and equals the oracle."""
    tr = synth.config_c3(0)[0]
    big = P.variants(capacity=80 * GiB)[3]
    _, so = O.replay(tr, big)
    rv = so["peak_reserved_vmm_bytes"]
    rs = so["peak_reserved_bytes"] - rv
    assert rv > 0 and rs > 0
    cap = max(rv, rs) + (min(rv, rs) // 2)          # each path fits, the sum does not
    pol = dict(big, capacity_bytes=cap, spool_max_inactive_bytes=cap)
    a, s, (n_split, n_rerun) = _run(R, [tr], [pol])
    assert n_rerun == 1 and n_split == 0
    _check_oracle([tr], [pol], a, s)


def test_split_oom_and_tight_capacity_fall_back(R):
    """Tight capacities (OOM in a path, BFC releases) on a latency batch:
    every unit equals the oracle, and some split units were re-run."""
    traces = [synth.random_trace(s, 400, 12, sizes=[1, 511, 300 * 1024, 1536 * 1024, 2 * MiB, 3 * MiB, 6 * MiB,
                                                    14 * MiB, 40 * MiB]) for s in range(6)]
    pols = P.variants(capacity=64 * MiB)
    for p in pols[2:]:
        p["frag_limit_bytes"] = 6 * MiB
    a, s, (n_split, n_rerun) = _run(R, traces, pols)
    assert n_rerun > 0 and n_split + n_rerun == 6 * len(traces)
    _check_oracle(traces, pols, a, s)


def test_split_invalid_trace_falls_back(R):
    """A malloc of a slot that is live on the OTHER path, and a free of a
    slot never allocated: no single path sees the error, the ledger warp
    does; the single-warp replay reports it (status INVALID at that event)."""
    bad1 = pack([("m", 0, 4 * MiB), ("m", 1, 1 * MiB), ("m", 0, 1024)])
    bad2 = pack([("m", 0, 4 * MiB), ("f", 0, 0), ("f", 7, 0)])
    pols = P.variants(capacity=1 * GiB)[2:4]
    for tr, at in ((bad1, 2), (bad2, 2)):
        _, s, (_, n_rerun) = _run(R, [tr], pols)
        assert n_rerun == len(pols)
        assert all(x["status"] == 1 and x["n_events_done"] == at for x in s[0]), s


def test_split_overflow_grows_class(R):
    """A split unit whose tables overflow re-runs in the next class (still
    split when that class has split instances) and equals the oracle."""
    tr = synth.config_c3(2)[0]
    pols = P.variants(capacity=80 * GiB)
    caps = np.full((len(pols), 4), 2, dtype=np.uint32)
    a, s, (n_split, _) = _run(R, [tr], pols, caps=caps)
    assert (caps > 2).any() and n_split > 0
    _check_oracle([tr], pols, a, s)


def test_path_units_throughput_placement(R):
    """More than 4 units per SM: GMLake units replay as path units (VMM path
    and small path in the two family launches, per-trace ledger, merge).
    Tight and loose capacities mix units that stay split, units the ledger
    demotes up front (requested bytes over capacity) and units the merge
    hands back (an OOM or release in a path, reserved sum over capacity);
    every record and statistic equals the oracle's."""
    sizes = [1, 511, 300 * 1024, 1536 * 1024, 2 * MiB, 3 * MiB, 6 * MiB, 14 * MiB, 40 * MiB]
    traces = [synth.random_trace(s, 300, 12, sizes=sizes) for s in range(80)]
    pols = P.variants(capacity=96 * MiB)
    for p in pols[2:]:
        p["frag_limit_bytes"] = 6 * MiB
    pols[3]["capacity_bytes"] = pols[3]["spool_max_inactive_bytes"] = 4 * GiB
    a, s, (n_split, n_rerun) = _run(R, traces, pols)
    assert len(traces) * len(pols) >= 4 * 148
    assert n_split > 0 and n_rerun > 0
    _check_oracle(traces, pols, a, s)
    a0, s0, _ = _run(R, traces, pols, no_split=True)
    assert np.array_equal(a0, a) and s0 == s


def test_path_units_ragged_and_invalid(R):
    """Throughput placement with empty traces, an invalid trace (malloc of a
    slot live on the other path) and OOM traces in the batch: the ledger
    demotes the invalid and certain-OOM units, empty traces merge to empty
    records, and every unit equals the oracle (status INVALID at the bad
    event for the invalid trace)."""
    sizes = [1, 300 * 1024, 2 * MiB, 3 * MiB, 6 * MiB, 14 * MiB, 40 * MiB]
    bad = pack([("m", 0, 4 * MiB), ("m", 1, 1 * MiB), ("m", 0, 1024)])
    traces = []
    for s in range(30):
        traces += [np.zeros(0, np.uint64), synth.random_trace(100 + s, 200, 10, sizes=sizes),
                   synth.random_trace(200 + s, 200, 40, sizes=[64 * MiB, 128 * MiB])]
    pols = P.variants(capacity=512 * MiB)
    for p in pols[2:]:
        p["frag_limit_bytes"] = 6 * MiB
    a, s, (n_split, _) = _run(R, traces + [bad], pols)
    assert (len(traces) + 1) * len(pols) >= 4 * 148 and n_split > 0
    _check_oracle(traces, pols, a, s)
    assert all(x["status"] == 1 and x["n_events_done"] == 2 for x in s[-1])
