"""Oracle vs the paper's definitions, by brute force after every event, plus
the closed-form no-new-peak theorem on every V3 trace."""
import numpy as np
import pytest

import oracle_lib as O
from invariants import Checker, theorem_holds
from tracegen import synth
from tracegen import policies as P

MiB = 1 << 20
GiB = 1 << 30
NO_BYTE_CAP = 1 << 62


def _variants(capacity, limit):
    base = dict(capacity=capacity, frag_limit=limit, spool_max_inactive_bytes=NO_BYTE_CAP)
    return {
        "gmlake": P.policy(P.GMLAKE, **base),
        "pfirst": P.policy(P.GMLAKE, P.F_S1_PBLOCK_FIRST, **base),
        "nocomp": P.policy(P.GMLAKE, P.F_NO_COMPANION, **base),
        "inval": P.policy(P.GMLAKE, P.F_SPLIT_INVALIDATES, **base),
        "remainder": P.policy(P.GMLAKE, P.F_REMAINDER_RULE, **base),
        "spool4": P.policy(P.GMLAKE, spool_max_entries=4, **base),
        "spool2_inval": P.policy(P.GMLAKE, P.F_SPLIT_INVALIDATES, spool_max_entries=2, **base),
        "gate": P.policy(P.GMLAKE, P.F_LIMIT_GATES_REQUEST, **base),
        "gate_inval": P.policy(P.GMLAKE, P.F_LIMIT_GATES_REQUEST | P.F_SPLIT_INVALIDATES, spool_max_entries=3, **base),
        "bytecap": P.policy(P.GMLAKE, capacity=capacity, frag_limit=limit, spool_max_inactive_bytes=8 * MiB),
        "bfc_torch": P.policy(P.BFC_TORCH, capacity=capacity),
        "bfc_exact": P.policy(P.BFC_EXACT, capacity=capacity),
    }


@pytest.mark.parametrize("name", list(_variants(1, 1)))
def test_fuzz_checked(name):
    """Random traces (mixed small-path and VMM sizes, tight capacity so that
    S5 and BFC release-and-retry fire) checked after every event."""
    n_ok = n_oom = 0
    for seed in range(12):
        cap = (24 + 8 * (seed % 4)) * 2 * MiB
        limit = [2 * MiB, 6 * MiB, 16 * MiB][seed % 3]
        pol = _variants(cap, limit)[name]
        sizes = [1, 300 * 1024, 1536 * 1024, 2 * MiB, 3 * MiB, 4 * MiB, 6 * MiB, 8 * MiB,
                 12 * MiB, 14 * MiB]
        ev = synth.random_trace(1000 + seed, 160, 10, sizes=sizes)
        st = Checker(pol).run(ev)
        n_ok += st["status"] == 0
        n_oom += st["status"] == 2
    assert n_ok > 0 and n_oom > 0     # both outcomes are checked two-way


@pytest.mark.parametrize("name", ["gmlake", "nocomp", "remainder", "bfc_torch", "bfc_exact", "spool4"])
def test_exhaustive_tiny_checked(name):
    """Every trace with 3 mallocs of 1..4 granules and every free
    interleaving (SURVEY §4 layer 3), capacity 6 granules so OOM fires."""
    for limit in (2 * MiB, 4 * MiB):
        pol = _variants(6 * 2 * MiB, limit)[name]
        for ev in synth.tiny_corpus(3, [2 * MiB, 4 * MiB, 6 * MiB, 8 * MiB]):
            Checker(pol).run(ev)


@pytest.mark.parametrize("flags", [0, P.F_S1_PBLOCK_FIRST, P.F_NO_COMPANION, P.F_SPLIT_INVALIDATES,
                                   P.F_REMAINDER_RULE, P.F_NO_COMPANION | P.F_SPLIT_INVALIDATES])
def test_theorem_no_new_peak(flags):
    """with limit = 1 chunk, 'each time the program reaches
    a new peak ... resulting in full memory utilization without
    fragmentation': reserved_vmm(t) = max_{t'<=t} active_vmm(t'), so the VMM
    utilization is exactly 1.0. Holds for every flag and every sPool cap."""
    for seed in range(40):
        cap = [8, 64][seed % 2]
        pol = P.policy(P.GMLAKE, flags, capacity=64 * GiB, frag_limit=2 * MiB,
                       spool_max_entries=cap, spool_max_inactive_bytes=[64 * GiB, 256 * MiB][seed % 2])
        sizes = None if seed % 3 else [2 * MiB, 6 * MiB, 10 * MiB, 64 * MiB, 1 * MiB]
        ev = synth.random_trace(seed, 600, 40, sizes=sizes, size_lo=1, size_hi=300 * MiB)
        _, st, tl = O.replay(ev, pol, timeline=True)
        assert st["status"] == 0
        assert theorem_holds(tl), seed
        assert st["peak_active_vmm_bytes"] == st["peak_reserved_vmm_bytes"]


def test_theorem_exhaustive_m4():
    """The theorem on all 26,880 traces of 4 mallocs x 1..4 granules."""
    pol = P.policy(P.GMLAKE, capacity=GiB, frag_limit=2 * MiB)
    n = 0
    for ev in synth.tiny_corpus(4, [2 * MiB, 4 * MiB, 6 * MiB, 8 * MiB]):
        _, st, tl = O.replay(ev, pol, timeline=True)
        assert theorem_holds(tl)
        assert st["final_active_bytes"] == 0          # I5: balanced -> nothing live
        n += 1
    assert n == 26880


def test_limit_is_not_free_lunch():
    """Fragmentation limit 128 MiB blocks splitting of
    small blocks, so reserved can exceed the running active max -- the
    theorem is specific to limit = 1 chunk (guards a no-op limit)."""
    ev = synth.lognormal_trace(5, 6, 60, 60 * MiB, sigma=0.8, extra_frac=0.3, interleave_frac=0.3)
    _, st, tl = O.replay(ev, P.policy(P.GMLAKE), timeline=True)
    assert not theorem_holds(tl)


def test_byte_cap_evicts_lru_inactive():
    """StitchFree (D17(ii)): when the inactive
    sBlocks hold more than the byte cap at malloc entry, the least recently
    used inactive ones are released -- never an active one -- and reserved
    memory is unchanged by the eviction."""
    pol = P.policy(P.GMLAKE, frag_limit=2 * MiB, spool_max_inactive_bytes=8 * MiB)
    ev = synth.lognormal_trace(9, 5, 30, 12 * MiB, sigma=0.7, lo=2 * MiB, hi=64 * MiB,
                               extra_frac=0.4, interleave_frac=0.4)
    c = Checker(pol)
    n_checked = 0
    for e in ev:
        pre = c.snap()
        status, rec = c.s.step(int(e))
        assert status == 0
        post = c.snap()
        post_ords = {b["ord"] for b in post["sb"]}
        gone = [b for b in pre["sb"] if b["ord"] not in post_ords]
        if gone:
            owned = set().union(*c.chunk_sets(pre).values()) if pre["h"] else set()
            inact = [b for b in pre["sb"]
                     if not any(ch in owned for lo, n in b["iv"] for ch in range(lo, lo + n))]
            assert all(b in inact for b in gone)
            lru = sorted(inact, key=lambda b: b["last_use"])[: len(gone)]
            assert sorted(b["ord"] for b in gone) == sorted(b["ord"] for b in lru)
            n_checked += 1
        if O.rec_fields(rec)["state"] not in (4, 7):
            assert post["c"]["reserved"] == pre["c"]["reserved"]
    assert n_checked > 0 and c.s.stats()["n_evict"] > 0


def test_balanced_traces_end_empty():
    """I5: every byte is freed at trace end (north_star invariant)."""
    for pol in P.variants(capacity=180 * GiB):
        ev = synth.lognormal_trace(3, 4, 80, 93e6, small_frac=0.2, extra_frac=0.2, interleave_frac=0.2)
        _, st = O.replay(ev, pol)
        assert st["status"] == 0 and st["final_active_bytes"] == 0
        assert st["peak_active_bytes"] <= st["peak_reserved_bytes"]
