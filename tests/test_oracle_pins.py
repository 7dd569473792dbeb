"""Pins of the CPU oracle against values the paper fixes (not against itself).

Each test names the passage it follows. Values here are hand-derived from the
paper (tests/golden/*.json carry their derivation) or closed forms.
"""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
from tracegen import pack, synth
from tracegen import policies as P

MiB = 1 << 20
GiB = 1 << 30
GOLD = Path(__file__).parent / "golden"


def _trace_mib(rows):
    return pack([(op, slot, size * MiB) for op, slot, size in rows])


def _f(r):
    return O.rec_fields(r)


# ---------------------------------------------------------------- fig:intro
def test_fig_intro_gmlake_stitches_block6():
    """'the VMS can map Block 6 to the Block 2 and 5 stitched
    block'. Hand trace: tests/golden/fig_intro.json."""
    g = json.loads((GOLD / "fig_intro.json").read_text())
    ev = _trace_mib(g["trace"])
    pol = P.policy(P.GMLAKE, capacity=g["capacity_mib"] * MiB,
                   frag_limit=g["gmlake"]["policy"]["frag_limit_mib"] * MiB)
    asg, st = O.replay(ev, pol)
    got = [[_f(a)["ord"], _f(a)["kind"], _f(a)["state"]] for a in asg]
    assert got == g["gmlake"]["records"]
    e = g["gmlake"]
    assert st["state_count"] == e["state_count"]
    for k in ("n_split", "n_stitch", "n_companion", "n_alloc", "vmm_calls", "oom_event"):
        assert st[k] == e[k], k
    assert st["peak_active_bytes"] == e["peak_active_mib"] * MiB
    assert st["peak_reserved_bytes"] == e["peak_reserved_mib"] * MiB
    # the stitched block of event 13 lives on Block 2's and Block 5's granules
    s = O.Stepper(pol)
    for i in range(14):
        s.step(ev[i])
    blk6 = [b for b in s.sblocks() if b["ord"] == g["gmlake"]["records"][13][0]][0]
    assert blk6["iv"] == [tuple(x) for x in g["gmlake"]["stitched_block6_intervals"]]


def test_fig_intro_bfc_cannot_hold_block6():
    """the splitting allocator 'cannot hold Block 6' and
    reports OOM."""
    g = json.loads((GOLD / "fig_intro.json").read_text())
    ev = _trace_mib(g["trace"])
    asg, st = O.replay(ev, P.policy(P.BFC_EXACT, capacity=g["capacity_mib"] * MiB))
    e = g["bfc_exact"]
    got = [[_f(a)["ord"], _f(a)["seg"], _f(a)["state"]] for a in asg[:13]]
    assert got == e["records"]
    assert st["oom_event"] == e["oom_event"] and st["status"] == 2
    assert _f(asg[13])["state"] == 5 and _f(asg[13])["ord"] == 0xFFFFFFFF
    assert all(a == 0 for a in asg[14:])
    assert st["peak_active_bytes"] == e["peak_active_mib"] * MiB
    assert st["peak_reserved_bytes"] == e["peak_reserved_mib"] * MiB


# ----------------------------------------------------- Algorithm 1 examples
UNIT = 100 * MiB   # SPEC.md L265-267 works in units of 100 MB; chunk = 1 unit


def _alg1_pol(**kw):
    return P.policy(P.GMLAKE, chunk=UNIT, small_threshold=UNIT, frag_limit=UNIT,
                    capacity=1000 * UNIT, **kw)


def _pool_400_200():
    # two S4 pBlocks of 4 and 2 units, then both freed: pPool {400, 200}
    return [("m", 0, 4 * UNIT), ("m", 1, 2 * UNIT), ("f", 0, 0), ("f", 1, 0)]


def test_alg1_single_block_s2():
    """size 300, pPool {400, 200} -> (2, [400])."""
    ev = pack(_pool_400_200() + [("m", 2, 3 * UNIT)])
    s = O.Stepper(_alg1_pol())
    for e in ev:
        _, a = s.step(e)
    assert _f(a)["state"] == 2 and _f(a)["kind"] == 0
    pb = {r[0]: r for r in s.pblocks()}
    F = pb[_f(a)["ord"]]
    assert (F[1], F[2]) == (0, 3)              # front 3 units of the 400 block (lo 0)
    assert sorted((r[2]) for r in pb.values()) == [1, 2, 3]


def test_alg1_multiple_blocks_s3():
    """size 500, pPool {400, 200} -> (3, [400, 200]); the last
    candidate is split to 100 (D14)."""
    ev = pack(_pool_400_200() + [("m", 2, 5 * UNIT)])
    s = O.Stepper(_alg1_pol())
    for e in ev:
        _, a = s.step(e)
    assert _f(a)["state"] == 3 and _f(a)["kind"] == 1
    sb = {b["ord"]: b for b in s.sblocks()}[_f(a)["ord"]]
    assert sb["size"] == 5 and sb["iv"] == [(0, 4), (4, 1)]


def test_alg1_insufficient_s4():
    """size 700 -> (4, [400, 200]); Alloc of the 100 shortfall."""
    ev = pack(_pool_400_200() + [("m", 2, 7 * UNIT)])
    s = O.Stepper(_alg1_pol())
    for e in ev:
        _, a = s.step(e)
    assert _f(a)["state"] == 4 and _f(a)["kind"] == 1
    sb = {b["ord"]: b for b in s.sblocks()}[_f(a)["ord"]]
    assert sb["iv"] == [(0, 4), (4, 2), (6, 1)]
    assert s.counters()["reserved"] == 7 * UNIT


def test_alg1_exact_sblock_s1():
    """SPEC.md L265 / PAPER.md L460: an exact-size inactive sBlock is returned
    in S1 ('the sole situation where an sBlock can be assigned')."""
    rows = [("m", 0, 4 * UNIT), ("m", 1, 2 * UNIT), ("m", 2, 1 * UNIT), ("m", 3, 2 * UNIT),
            ("f", 2, 0), ("f", 3, 0), ("m", 4, 3 * UNIT), ("f", 4, 0), ("f", 0, 0), ("f", 1, 0),
            ("m", 5, 3 * UNIT)]
    ev = pack(rows)
    asg, st = O.replay(ev, _alg1_pol())
    assert _f(asg[6])["state"] == 3 and _f(asg[6])["kind"] == 1
    assert _f(asg[10]) == dict(ord=_f(asg[6])["ord"], kind=1, state=1, seg=0)
    # sPool-first reading D5 vs its variant: with S1_PBLOCK_FIRST there is no
    # 3-unit pBlock either, so the same sBlock is returned
    asg2, _ = O.replay(ev, _alg1_pol(flags=P.F_S1_PBLOCK_FIRST))
    assert _f(asg2[10])["kind"] == 1


def test_s2_tie_highest_ordinal():
    """Alg. 1 L6-8 replaces CB on every block >= bSize, so
    among equal-size best fits the LAST in pool order wins (D6)."""
    rows = [("m", 0, 4 * UNIT), ("m", 1, 4 * UNIT), ("m", 2, 4 * UNIT),
            ("f", 0, 0), ("f", 1, 0), ("f", 2, 0), ("m", 3, 1 * UNIT)]
    s = O.Stepper(_alg1_pol())
    for e in pack(rows):
        _, a = s.step(e)
    pb = {r[0]: r for r in s.pblocks()}
    assert pb[_f(a)["ord"]][1] == 8           # carved from the third block (lo 8)


# ----------------------------------------------------------------- Stitch
def test_stitch_1g_2g_adds_no_memory():
    """p1 (1 GB) + p2 (2 GB) stitched into a 3 GB sBlock;
    sBlocks 'never create cuMemCreate new physical chunks'."""
    rows = [("m", 0, 1 * GiB), ("m", 1, 2 * GiB), ("f", 0, 0), ("f", 1, 0), ("m", 2, 3 * GiB)]
    s = O.Stepper(P.policy(P.GMLAKE))
    for e in pack(rows[:4]):
        s.step(e)
    before = s.stats()["vmm_calls"][1], s.counters()["reserved"]
    _, a = s.step(pack(rows[4:])[0])
    assert _f(a)["state"] == 3 and _f(a)["kind"] == 1
    sb = {b["ord"]: b for b in s.sblocks()}[_f(a)["ord"]]
    assert sb["size"] * 2 * MiB == 3 * GiB
    assert sum(n for _, n in sb["iv"]) == sb["size"]
    assert (s.stats()["vmm_calls"][1], s.counters()["reserved"]) == before == (1536, 3 * GiB)


# ------------------------------------------------------------------ Table 1
TABLE1_2MB = dict(reserve=0.003, create=18.1, map=0.70, access=96.8, total=115.4)


def test_table1_call_counts():
    """'one cuMemAddressReserve but multiple cuMemCreate,
    cuMemMap, and cuMemSetAccess for each physical chunk'; a 2 GB Alloc in
    2 MB chunks costs 115.4 cudaMalloc units (Table 1)."""
    _, st = O.replay(pack([("m", 0, 2 * GiB)]), P.policy(P.GMLAKE))
    assert st["vmm_calls"][:4] == [1, 1024, 1024, 1024]
    n = st["vmm_calls"]
    cost = (n[0] * TABLE1_2MB["reserve"] + n[1] * TABLE1_2MB["create"] / 1024
            + n[2] * TABLE1_2MB["map"] / 1024 + n[3] * TABLE1_2MB["access"] / 1024)
    # the printed column sums to 115.603; the printed total is 115.4 (<1%)
    assert abs(cost / TABLE1_2MB["total"] - 1) < 0.01


# ------------------------------------------------------------- convergence
def _states(asg):
    return [_f(a)["state"] for a in asg]


def test_convergence_companion():
    """after a few iterations only S1 is used; the
    companion sBlock of a split is reused as an exact match."""
    it = [("m", "a", 4), ("f", "a", 0), ("m", "b", 2), ("m", "c", 2), ("f", "b", 0), ("f", "c", 0)]
    ev = synth.periodic([(op, n, sz * 2 * MiB) for op, n, sz in it], 4)
    pol = P.policy(P.GMLAKE, frag_limit=2 * MiB)
    asg, _ = O.replay(ev, pol)
    st = _states(asg)
    assert [st[i] for i in (0, 2, 3)] == [4, 2, 1]
    assert _f(asg[6])["kind"] == 1 and st[6] == 1          # iteration 2: a -> sBlock s0
    assert all(st[i] == 1 for i in range(6, 24) if _f(asg[i])["state"] != 0)
    asg2, _ = O.replay(ev, P.policy(P.GMLAKE, P.F_NO_COMPANION, frag_limit=2 * MiB))
    st2 = _states(asg2)
    assert st2[6] == 3                                     # stitched in iteration 2
    assert all(st2[i] == 1 for i in range(12, 24) if st2[i] != 0)


def test_convergence_s4_stitch():
    """{a=3; b=5; free a; c=4; free b; free c}: c -> S4 stitch
    of P0 with a 1-granule Alloc; reserved == active then."""
    it = [("m", "a", 3), ("m", "b", 5), ("f", "a", 0), ("m", "c", 4), ("f", "b", 0), ("f", "c", 0)]
    ev = synth.periodic([(op, n, sz * 2 * MiB) for op, n, sz in it], 3)
    asg, st, tl = O.replay(ev, P.policy(P.GMLAKE, frag_limit=2 * MiB), timeline=True)
    s = _states(asg)
    assert [s[0], s[1], s[3]] == [4, 4, 4] and _f(asg[3])["kind"] == 1
    assert tl[3][1] == tl[3][0] == 9 * 2 * MiB
    assert all(s[i] in (0, 1) for i in range(6, 18))


# ------------------------------------------------------------------ metrics
def test_metric_identities():
    """utilization = peak active / peak reserved,
    fragmentation = 1 - utilization, MemReductionRatio over sums."""
    from oracle import metrics as M
    assert M.utilization(72, 80) == pytest.approx(0.9)
    assert M.utilization(0, 0) == 1.0
    assert M.utilization(72, 80) + M.fragmentation(72, 80) == 1.0
    assert M.mem_reduction_ratio([80, 20], [60, 20]) == pytest.approx(0.2)
    assert M.mem_reduction_ratio([100], [75]) == pytest.approx(0.25)
    with pytest.raises(ValueError):
        M.mem_reduction_ratio([1], [1, 2])


def test_convergence_analysis_matches_hand_examples():
    """f4's analysis (paper_2401_08156_b200.analysis, host arithmetic on
    records) on the App. B examples: stable from iteration 1 with the
    companion (iteration 0 splits), from iteration 2 without it (iteration 1
    stitches)."""
    from paper_2401_08156_b200 import analysis as An
    it = [("m", "a", 4), ("f", "a", 0), ("m", "b", 2), ("m", "c", 2), ("f", "b", 0), ("f", "c", 0)]
    ev = synth.periodic([(op, n, sz * 2 * MiB) for op, n, sz in it], 4)
    starts = [6 * i for i in range(4)]
    asg, _ = O.replay(ev, P.policy(P.GMLAKE, frag_limit=2 * MiB))
    h = An.state_histograms(asg, starts)
    assert h.shape == (4, 7) and list(h[0][:4]) == [1, 1, 0, 1] and An.stable_after(h) == 1
    asg2, _ = O.replay(ev, P.policy(P.GMLAKE, P.F_NO_COMPANION, frag_limit=2 * MiB))
    h2 = An.state_histograms(asg2, starts)
    assert h2[1][2] == 1 and An.stable_after(h2) == 2
    _, _, tl = O.replay(ev, P.policy(P.GMLAKE, frag_limit=2 * MiB), timeline=True)
    pk = An.iteration_peaks(tl[:, :2], starts)
    assert pk.shape == (4, 2) and all(pk[:, 1] == 4 * 2 * MiB)


# ------------------------------------------------------- D21 / BFC goldens
def _bfc_pol(kind, cap=80 * GiB):
    return {"bfc_torch": P.policy(P.BFC_TORCH, capacity=cap), "bfc_exact": P.policy(P.BFC_EXACT, capacity=cap),
            "gmlake": P.policy(P.GMLAKE, capacity=cap)}[kind]


def test_bfc_d21_thresholds():
    """D21 (PyTorch's caching allocator, the baseline of PAPER.md L624; BFC
    ops of L116-125): segment sizes and split decisions at every threshold,
    hand-derived in tests/golden/bfc_d21.json."""
    g = json.loads((GOLD / "bfc_d21.json").read_text())["single_malloc"]
    for kind, raw, state, reserved, active, nblocks in g["cases"]:
        s = O.Stepper(_bfc_pol(kind))
        status, a = s.step(int(pack([("m", 0, raw)])[0]))
        assert status == 0 and _f(a)["state"] == int(state), (kind, raw)
        c = s.counters()
        assert (c["reserved"], c["active"]) == (reserved, active), (kind, raw, c)
        assert len(s.bfc()) == nblocks, (kind, raw)


def test_bfc_release_and_retry():
    """PyTorch's OOM path (D21): when a new segment does not fit, every fully
    free segment is released and the allocation retried once; OOM only if it
    still does not fit (tests/golden/bfc_d21.json, release_retry)."""
    g = json.loads((GOLD / "bfc_d21.json").read_text())["release_retry"]
    asg, st = O.replay(_trace_mib(g["trace"]), P.policy(P.BFC_TORCH, capacity=g["capacity_mib"] * MiB))
    got = [[_f(a)["ord"], _f(a)["seg"], _f(a)["state"]] for a in asg]
    assert got == g["records"]
    for k in ("n_seg_alloc", "n_seg_release", "oom_event"):
        assert st[k] == g[k], k
    assert st["peak_reserved_bytes"] == g["peak_reserved_mib"] * MiB
    assert st["peak_active_bytes"] == g["peak_active_mib"] * MiB


# ----------------------------------------------------- StitchFree goldens
def _units(rows, u=2 * MiB):
    return pack([(op, slot, n * u) for op, slot, n in rows])


def _sf_pol(flags=0, cap=4096):
    return P.policy(P.GMLAKE, flags, capacity=64 * 2 * MiB, frag_limit=2 * MiB, spool_max_entries=cap)


def _recs(asg):
    return [[_f(a)["ord"], _f(a)["kind"], _f(a)["state"]] for a in asg]


def _spool_after(ev, pol):
    s = O.Stepper(pol)
    for e in ev:
        s.step(int(e))
    return [b["ord"] for b in s.sblocks()], s.stats()


def test_stitchfree_count_cap_evicts_lru():
    """at the sPool cap StitchFree releases the
    LEAST recently used inactive sBlock (tests/golden/stitchfree.json)."""
    g = json.loads((GOLD / "stitchfree.json").read_text())["lru_count_cap"]
    ev, pol = _units(g["trace"]), _sf_pol(cap=g["spool_max_entries"])
    asg, st = O.replay(ev, pol)
    assert _recs(asg) == g["records"]
    order, st = _spool_after(ev, pol)
    assert order == g["spool_after"] and st["n_evict"] == g["n_evict"]


def test_stitchfree_spares_sblocks_of_this_malloc():
    """D17: the companion created by the split of this same malloc is not a
    count-cap victim; the allocation stitch goes over the (soft) cap."""
    g = json.loads((GOLD / "stitchfree.json").read_text())["born_exclusion"]
    ev, pol = _units(g["trace"]), _sf_pol(cap=g["spool_max_entries"])
    asg, _ = O.replay(ev, pol)
    assert _recs(asg) == g["records"]
    order, st = _spool_after(ev, pol)
    assert order == g["spool_after"]
    for k in ("n_evict", "n_companion", "n_stitch"):
        assert st[k] == g[k], k


def test_split_invalidates_victims():
    """D12 re-point (default) vs SPLIT_INVALIDATES: the sBlock
    over a split parent survives by default and is released by the variant."""
    g = json.loads((GOLD / "stitchfree.json").read_text())["split_invalidates"]
    ev = _units(g["trace"])
    asg, _ = O.replay(ev, _sf_pol())
    assert _recs(asg) == g["records_default"]
    assert _spool_after(ev, _sf_pol())[0] == g["spool_after_default"]
    asg2, st2 = O.replay(ev, _sf_pol(P.F_SPLIT_INVALIDATES))
    assert _recs(asg2) == g["records_default"]
    order, st = _spool_after(ev, _sf_pol(P.F_SPLIT_INVALIDATES))
    assert order == g["spool_after_invalidates"] and st["n_evict"] == 1


# ------------------------------------------- readings D16 and D8' (goldens)
def _gm_recs(asg):
    return [[_f(a)["ord"], _f(a)["kind"], _f(a)["state"]] for a in asg]


def _mib_f(rows):
    return pack([(op, slot, int(size * MiB)) for op, slot, size in rows])


def test_s5_after_small_path_release():
    """D16 (SPEC.md OOM last resort order): the small path's
    fully free segments are released before an Alloc is failed; S5 only if
    the shortfall still does not fit (tests/golden/gmlake_readings.json)."""
    G = json.loads((GOLD / "gmlake_readings.json").read_text())
    for name in ("d16_release_then_alloc", "d16_still_oom"):
        g = G[name]
        pol = P.policy(P.GMLAKE, capacity=g["capacity_mib"] * MiB, frag_limit=g["frag_limit_mib"] * MiB)
        asg, st = O.replay(_mib_f(g["trace"]), pol)
        assert _gm_recs(asg) == g["records"], name
        assert st["status"] == g["status"] and st["n_seg_release"] == g["n_seg_release"], name
        if "peak_reserved_mib" in g:
            assert st["peak_reserved_bytes"] == g["peak_reserved_mib"] * MiB
            assert st["final_reserved_bytes"] == g["final_reserved_mib"] * MiB
        if "oom_event" in g:
            assert st["oom_event"] == g["oom_event"]


def test_limit_gates_request():
    """D8' (PAPER.md L571 read for the request, L322): with
    LIMIT_GATES_REQUEST a tensor below the fragmentation limit takes the small
    path; without it (literal D8) it takes the VMM path."""
    g = json.loads((GOLD / "gmlake_readings.json").read_text())["d8_gate"]
    ev = _mib_f(g["trace"])
    kw = dict(capacity=g["capacity_mib"] * MiB, frag_limit=g["frag_limit_mib"] * MiB)
    asg, st = O.replay(ev, P.policy(P.GMLAKE, P.F_LIMIT_GATES_REQUEST, **kw))
    assert _gm_recs(asg) == g["records_gate"] and [_f(a)["seg"] for a in asg] == g["seg_gate"]
    assert st["peak_reserved_bytes"] == g["peak_reserved_mib_gate"] * MiB
    asg, st = O.replay(ev, P.policy(P.GMLAKE, **kw))
    assert _gm_recs(asg) == g["records_literal"]
    assert st["peak_reserved_bytes"] == g["peak_reserved_mib_literal"] * MiB


def test_product_policy_report_metrics():
    """The product's host finalize (analysis.policy_report) follows PAPER.md
    L629-635: MemReductionRatio([80, 20], [60, 20]) = 0.2,
    utilization = sum peak active / sum peak reserved."""
    from paper_2401_08156_b200 import analysis as An
    assert An.mem_reduction_ratio([80, 20], [60, 20]) == pytest.approx(0.2)

    def st(a, q, r, status=0):
        return dict(peak_active_bytes=a, peak_requested_bytes=q, peak_reserved_bytes=r, status=status)
    rep = An.policy_report([[st(70, 60, 80), st(72, 70, 72)], [st(10, 10, 20), st(18, 18, 20)],
                            [st(5, 5, 10), st(0, 0, 0, status=2)]])
    assert rep["V0"]["utilization"] == pytest.approx(85 / 110)
    assert rep["V1"]["mem_reduction_vs_V0"] == pytest.approx((100 - 92) / 100)
    assert rep["V1"]["matched_traces"] == 2 and rep["V1"]["oom_traces"] == 1
    assert rep["V0"]["utilization_requested"] == pytest.approx(75 / 110)
