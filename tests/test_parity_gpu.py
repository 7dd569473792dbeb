"""Parity of the CUDA replay (K1 via the C ABI) with the CPU oracle:
bit-exact on every assignment record and every statistic (integer work).

Inputs span the paper-shaped configurations (C1 fig:intro, C2 OPT-1.3B, C3
GPT-NeoX-20B ZeRO-3 ranks, a C4 sample), the irregular SPEC corpus, fuzz
traces with tight capacities (OOM paths), the exhaustive tiny corpus, ragged
batches with empty traces, forced table overflow (re-run path) and the
global-memory arena path.
"""
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


def _compare(R, traces, pols, caps=None, check_asg=True, sample_every=1):
    import torch
    batch = R.upload(traces)
    # sentinel fill: every record (incl. the zeros after a terminating event) must come from K1
    sent = torch.full((len(pols), max(batch.total, 1)), -1, dtype=torch.int64, device="cuda") if check_asg else None
    asg, st = R.run(batch, pols, with_assignments=check_asg, caps=caps, assignments=sent)
    torch.cuda.synchronize()
    stats = R.decode_stats(st, len(traces), len(pols))
    a = asg.cpu().numpy().view(np.uint64) if check_asg else None
    off = 0
    n_cmp = 0
    for t, tr in enumerate(traces):
        if t % sample_every == 0:
            for p, pol in enumerate(pols):
                ao, so = O.replay(tr, pol)
                g = stats[t][p]
                assert g == so, (t, p, {k: (g[k], so[k]) for k in so if g[k] != so[k]})
                if check_asg:
                    got = a[p, off:off + len(tr)]
                    if not np.array_equal(got, ao):
                        i = int(np.nonzero(got != ao)[0][0])
                        raise AssertionError(f"trace {t} policy {p} event {i}: "
                                             f"{O.rec_fields(got[i])} != {O.rec_fields(ao[i])}")
                n_cmp += 1
        off += len(tr)
    return stats, n_cmp


def _compare_all(R, traces, pols, caps=None):
    """Every (trace, policy) unit against the oracle, element by element;
    the oracle replays run on all host cores (threads: the ctypes call
    releases the GIL). Returns the GPU stats."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    import torch
    batch = R.upload(traces)
    sent = torch.full((len(pols), max(batch.total, 1)), -1, dtype=torch.int64, device="cuda")
    asg, st = R.run(batch, pols, caps=caps, assignments=sent)
    torch.cuda.synchronize()
    stats = R.decode_stats(st, len(traces), len(pols))
    a = asg.cpu().numpy().view(np.uint64)
    offs = np.concatenate([[0], np.cumsum([len(t) for t in traces])])

    def job(tp):
        t, p = tp
        ao, so = O.replay(traces[t], pols[p])
        g = stats[t][p]
        if g != so:
            return f"trace {t} policy {p} stats: " + str({k: (g[k], so[k]) for k in so if g[k] != so[k]})
        got = a[p, offs[t]:offs[t + 1]]
        if not np.array_equal(got, ao):
            i = int(np.nonzero(got != ao)[0][0])
            return f"trace {t} policy {p} event {i}: {O.rec_fields(got[i])} != {O.rec_fields(ao[i])}"
        return None

    pairs = [(t, p) for t in range(len(traces)) for p in range(len(pols))]
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        bad = [m for m in ex.map(job, pairs, chunksize=64) if m]
    assert not bad, (len(bad), bad[:5])
    return stats


def test_fig_intro_all_variants(R):
    pols = P.variants(capacity=24 * MiB)
    for p in pols:
        p["frag_limit_bytes"] = 2 * MiB
    stats, _ = _compare(R, [synth.fig_intro()], pols)
    assert stats[0][1]["oom_event"] == 13            # BFC cannot hold Block 6
    assert stats[0][2]["status"] == 0                 # GMLake stitches it


def test_fuzz_tight_capacity(R):
    traces = [synth.random_trace(s, 300, 12, sizes=[1, 511, 513, 300 * 1024, 1536 * 1024, 2 * MiB,
                                                    3 * MiB, 6 * MiB, 14 * MiB, 40 * MiB])
              for s in range(24)]
    for cap_mib in (48, 96, 4096):
        pols = P.variants(capacity=cap_mib * MiB)
        for p in pols[2:]:
            p["frag_limit_bytes"] = [2 * MiB, 6 * MiB, 16 * MiB][cap_mib % 3]
        pols[7]["spool_max_entries"] = 3
        pols.append(P.policy(P.GMLAKE, P.F_S1_PBLOCK_FIRST | P.F_NO_COMPANION, capacity=cap_mib * MiB,
                             frag_limit=4 * MiB, spool_max_inactive_bytes=16 * MiB))
        _compare(R, traces, pols)


def test_tiny_corpus(R):
    traces = list(synth.tiny_corpus(3, [2 * MiB, 4 * MiB, 6 * MiB, 8 * MiB]))
    pols = P.variants(capacity=12 * MiB)
    for p in pols[2:]:
        p["frag_limit_bytes"] = 4 * MiB
    pols[3]["frag_limit_bytes"] = 2 * MiB
    _compare(R, traces, pols)


def _tiny_pols():
    pols = P.variants(capacity=12 * MiB)
    for p in pols[2:]:
        p["frag_limit_bytes"] = 4 * MiB
    pols[3]["frag_limit_bytes"] = 2 * MiB
    return pols


def test_tiny_corpus_m4_exhaustive(R):
    """every m = 4 trace (4 sizes, every free interleaving:
    26,880 traces x 8 policies), each unit element by element."""
    traces = list(synth.tiny_corpus(4, [2 * MiB, 4 * MiB, 6 * MiB, 8 * MiB]))
    assert len(traces) == 26880
    _compare_all(R, traces, _tiny_pols())


def test_tiny_corpus_m5_sample(R):
    """m = 5 (967,680 traces): every 61st trace (15,864 x 8 policies)."""
    import itertools
    traces = list(itertools.islice(synth.tiny_corpus(5, [2 * MiB, 4 * MiB, 6 * MiB, 8 * MiB]), 0, None, 61))
    assert len(traces) == 15864
    _compare_all(R, traces, _tiny_pols())


def test_ragged_batch_with_empty_traces(R):
    traces = [np.zeros(0, np.uint64), synth.fig_intro(), np.zeros(0, np.uint64),
              pack([("m", 0, 5)]), synth.random_trace(9, 1000, 50, size_lo=1, size_hi=300 * MiB)]
    _compare(R, traces, P.variants(capacity=4 * GiB))


def test_extreme_sizes(R):
    traces = [pack([("m", 0, (1 << 40) - 1), ("m", 1, 1)]),
              pack([("m", 0, 1), ("m", 1, 2 * MiB - 1), ("m", 2, 2 * MiB), ("f", 1, 0), ("m", 1, 1 * MiB + 1)])]
    _compare(R, traces, P.variants(capacity=80 * GiB))


def test_irregular_corpus(R):
    traces = [synth.lognormal_trace(s, 3, 46 if s % 2 else 76, 93e6 if s % 2 else 85e6,
                                    extra_frac=0.1 * (s % 4), interleave_frac=0.1 * (s % 3),
                                    small_frac=0.05 * (s % 5))
              for s in range(50)]
    _compare(R, traces, P.variants(capacity=80 * GiB))


def test_overflow_rerun_matches(R):
    """D30: table capacity never changes a result -- forced tiny tables
    overflow, are re-run with larger ones, and still match."""
    traces = [synth.lognormal_trace(7, 3, 60, 40e6, extra_frac=0.3, interleave_frac=0.3, small_frac=0.2)]
    pols = P.variants(capacity=80 * GiB)
    caps = np.full((len(traces) * len(pols), 4), 2, dtype=np.uint32)
    _compare(R, traces, pols, caps=caps)
    assert (caps > 2).any()


def test_global_arena_path(R):
    """Units whose tables exceed shared memory run on a global-memory arena."""
    traces = [synth.random_trace(11, 2000, 80, size_lo=1, size_hi=200 * MiB)]
    pols = P.variants(capacity=80 * GiB)
    caps = np.full((len(pols), 4), 20000, dtype=np.uint32)
    _compare(R, traces, pols, caps=caps)


def test_c2_opt13b_full(R):
    ev, _ = synth.config_c2()
    _compare(R, [ev], P.variants(capacity=80 * GiB))


def test_c3_neox_ranks(R):
    traces = [synth.config_c3(r)[0] for r in range(8)]
    _compare(R, traces, P.variants(capacity=80 * GiB))


def test_c4_sample(R):
    idx = [0, 511, 1024, 1777, 2600, 3333, 3500, 4095]
    traces = [synth.config_c4(i)[0] for i in idx]
    _compare(R, traces, P.variants(capacity=180 * GiB))


def test_invalid_trace_flags(R):
    import torch
    bad = pack([("m", 0, 4 * MiB)]).tolist() + [int(pack([("f", 1, 0)])[0])]
    batch = R.upload([np.array(bad, dtype=np.uint64)])
    _, st = R.run(batch, P.variants()[:3])
    torch.cuda.synchronize()
    s = R.decode_stats(st, 1, 3)
    assert all(x["status"] == 1 and x["n_events_done"] == 1 for x in s[0])


def test_timeline_matches_oracle(R):
    """f4: the optional (active, reserved) per-event series equals the
    oracle's, including the terminating OOM event and zeros after it."""
    import torch
    traces = [synth.fig_intro(), synth.random_trace(5, 400, 12, sizes=[1, 300 * 1024, 2 * MiB, 6 * MiB, 14 * MiB]),
              synth.config_c2()[0]]
    pols = P.variants(capacity=48 * MiB)
    for p in pols[2:]:
        p["frag_limit_bytes"] = 2 * MiB
    for tr, pl in ((traces[0], pols), (traces[1], pols), (traces[2], P.variants(capacity=80 * GiB))):
        batch = R.upload([tr])
        # sentinel fill: the zeros after a terminating event must be written by K1
        tl = torch.full((len(pl), len(tr), 2), -1, dtype=torch.int64, device="cuda")
        asg, st = R.run(batch, pl, timeline=tl)
        torch.cuda.synchronize()
        got = tl.cpu().numpy().view(np.uint64)
        for p, pol in enumerate(pl):
            _, _, tlo = O.replay(tr, pol, timeline=True)
            assert np.array_equal(got[p], tlo[:, :2]), p


def test_convergence_on_c2_matches_oracle(R):
    """f4: per-iteration S-state histograms and 'stable after k iterations'
    from the GPU records equal the oracle's."""
    from paper_2401_08156_b200 import analysis as An
    ev, starts = synth.config_c2()
    pols = P.variants(capacity=80 * GiB)
    batch = R.upload([ev])
    asg, _ = R.run(batch, pols)
    import torch
    torch.cuda.synchronize()
    a = asg.cpu().numpy().view(np.uint64)
    for p, pol in enumerate(pols):
        h = An.state_histograms(a[p], starts)
        ho = An.state_histograms(O.replay(ev, pol)[0], starts)
        assert np.array_equal(h, ho)
        if p == 2:   # GMLake default: only S1 on the VMM path from iteration 2 on
            assert An.stable_after(h) == 2, h[:5]


def test_c4_bench_configuration_full(R):
    """C4 at the size and in the launch configuration bench.py times (512
    traces x 8 policies per GPU = 4096 units: throughput mode, global-memory
    arenas, 4 warps per CTA, classes launched concurrently, table hints from
    a previous replay as in the timed steps): EVERY (trace, policy) unit's
    records and stats are bit-exact against the oracle (oracle on all host
    cores), and every unit's invariants hold."""
    import os
    import bench
    os.environ["GML_C4_PER_GPU"] = "512"
    W = bench.Workload("c4", 1)
    traces, pols = W.load(list(range(W.n))), W.pols
    assert len(traces) == 512
    # the timed steps' table hints: the classes a first replay of the batch
    # ended in (gml_replay writes them back into caps)
    batch = R.upload(traces)
    caps = np.zeros((len(traces) * len(pols), 4), dtype=np.uint32)
    R.run(batch, pols, with_assignments=False, caps=caps)
    assert caps.any()
    del batch
    stats = _compare_all(R, traces, pols, caps=caps)
    for per_t in stats:
        for s in per_t:
            assert s["n_events_done"] == s["n_events"] or s["status"] == 2
            assert s["peak_active_bytes"] <= s["peak_reserved_bytes"]


def test_largest_class_70k_pblocks(R):
    """D30 at the top of the class ladder: 70,000 live 2 MiB tensors in a
    180 GiB pool need 70,000 pBlocks, more than class C9 holds; the unit
    overflows up the ladder to C10 and still matches the oracle."""
    from tracegen import SlotAssigner
    sa = SlotAssigner()
    for i in range(70000):
        sa.malloc(i, 2 * MiB)
    for i in range(0, 70000, 7):
        sa.free(i)
    for i in range(0, 70000, 7):
        sa.malloc(("b", i), 2 * MiB)
    ev = np.array(sa.events, dtype=np.uint64)
    pols = [P.policy(P.GMLAKE, capacity=180 * GiB, frag_limit=2 * MiB), P.policy(P.BFC_TORCH, capacity=180 * GiB)]
    stats, _ = _compare(R, [ev], pols)
    assert stats[0][0]["max_pblocks"] == 70000


def _random_policy(rng):
    """A random point of the policy space: kind, every ambiguity flag,
    fragmentation limit, sPool caps, capacity and chunk size."""
    kind = [P.BFC_TORCH, P.BFC_EXACT, P.GMLAKE, P.GMLAKE, P.GMLAKE][rng.integers(5)]
    flags = int(rng.integers(32)) if kind == P.GMLAKE else 0
    cap = int([96, 512, 2048, 8192, 8192][rng.integers(5)]) * MiB
    chunk = int([2, 2, 2, 4, 1][rng.integers(5)]) * MiB
    return P.policy(kind, flags, capacity=cap, chunk=chunk,
                    frag_limit=int([2, 4, 6, 16, 64, 128][rng.integers(6)]) * MiB,
                    spool_max_entries=int([1, 2, 3, 8, 64, 4096][rng.integers(6)]),
                    spool_max_inactive_bytes=[0, 16 * MiB, None][rng.integers(3)])


def test_random_policy_space_fuzz(R):
    """Fuzz over the whole policy space (random kind / flag set / limit /
    caps / capacity / chunk size) x 2,000 random and irregular traces, on
    the throughput (global-arena) placement: every unit element by element
    against the oracle."""
    rng = np.random.default_rng(20260317)
    pols = [_random_policy(rng) for _ in range(16)]
    sizes = [1, 511, 513, 300 * 1024, 1 * MiB, 1536 * 1024, 2 * MiB, 3 * MiB, 6 * MiB, 14 * MiB, 40 * MiB,
             130 * MiB]
    traces = []
    for s in range(2000):
        if s % 4 == 3:
            traces.append(synth.lognormal_trace(s, 2, 12 + s % 20, 20e6, extra_frac=0.2, interleave_frac=0.2,
                                                small_frac=0.3))
        elif s % 4 == 2:
            traces.append(synth.random_trace(s, 100 + s % 400, 4 + s % 30, sizes=sizes))
        else:
            traces.append(synth.random_trace(s, 100 + s % 400, 4 + s % 30, size_lo=1, size_hi=200 * MiB,
                                             balanced=bool(s % 2)))
    stats = _compare_all(R, traces, pols)
    ooms = sum(1 for per_t in stats for x in per_t if x["status"] == 2)
    assert 0 < ooms < len(traces) * len(pols)         # both the OOM paths and complete replays are covered
