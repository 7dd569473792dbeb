"""The PRODUCT allocation engine (paper_2401_08156_b200/csrc/policy.cuh)
compiled for the CPU and compared with the oracle, record by record and stat
by stat, without a GPU:

* width 1  -- the HostWarp executor the live allocator runs;
* width 32 -- SimWarp, 32 threads emulating the lanes of one warp, running
  the kernel's lane-parallel code paths (k-ary searches, PIN bit shifts,
  per-interval ownership with atomics, vector free-list scans) with every
  ballot / shuffle / __syncwarp as a barrier exchange. This is what caught
  the two leader-write races (H[slot], the BFC free-row link) that only a
  warp could hit.

The GPU parity tests (test_parity_gpu.py) check the same engine inside K1.
"""
import numpy as np
import pytest

import engine_lib as E
import oracle_lib as O
from tracegen import pack, synth
from tracegen import policies as P

MiB = 1 << 20
GiB = 1 << 30


def _compare(traces, pols, width):
    for t, tr in enumerate(traces):
        for p, pol in enumerate(pols):
            a, s, ovf = E.replay(tr, pol, width)
            ao, so = O.replay(tr, pol)
            assert ovf == 0, (t, p, ovf)
            if not np.array_equal(a, ao):
                i = int(np.nonzero(a != ao)[0][0])
                raise AssertionError(f"width {width} trace {t} policy {p} event {i}: "
                                     f"{O.rec_fields(a[i])} != {O.rec_fields(ao[i])}")
            assert s == so, (width, t, p, {k: (s[k], so[k]) for k in so if s[k] != so[k]})


def _fuzz_pols(cap_mib):
    pols = P.variants(capacity=cap_mib * MiB)
    for p in pols[2:]:
        p["frag_limit_bytes"] = [2 * MiB, 6 * MiB, 16 * MiB][cap_mib % 3]
    pols[7]["spool_max_entries"] = 3
    pols.append(P.policy(P.GMLAKE, P.F_S1_PBLOCK_FIRST | P.F_NO_COMPANION, capacity=cap_mib * MiB,
                         frag_limit=4 * MiB, spool_max_inactive_bytes=16 * MiB))
    return pols


FUZZ_SIZES = [1, 511, 513, 300 * 1024, 1536 * 1024, 2 * MiB, 3 * MiB, 6 * MiB, 14 * MiB, 40 * MiB]


@pytest.mark.parametrize("width", [1, 32])
def test_fig_intro(width):
    pols = P.variants(capacity=24 * MiB)
    for p in pols:
        p["frag_limit_bytes"] = 2 * MiB
    _compare([synth.fig_intro()], pols, width)


@pytest.mark.parametrize("width", [1, 32])
def test_fuzz_tight_capacity(width):
    """OOM / release-and-retry / LRU caps / every flag, capacities 48 MiB-4 GiB."""
    n = 24 if width == 1 else 8
    traces = [synth.random_trace(s, 300, 12, sizes=FUZZ_SIZES) for s in range(n)]
    for cap in (48, 96, 4096):
        _compare(traces, _fuzz_pols(cap), width)


@pytest.mark.parametrize("width", [1, 32])
def test_tiny_corpus(width):
    traces = list(synth.tiny_corpus(3, [2 * MiB, 4 * MiB, 6 * MiB, 8 * MiB]))
    if width == 32:
        traces = traces[::7]
    pols = P.variants(capacity=12 * MiB)
    for p in pols[2:]:
        p["frag_limit_bytes"] = 4 * MiB
    pols[3]["frag_limit_bytes"] = 2 * MiB
    _compare(traces, pols, width)


@pytest.mark.parametrize("width", [1, 32])
def test_irregular_corpus(width):
    seeds = range(50) if width == 1 else range(0, 50, 10)
    traces = [synth.lognormal_trace(s, 3, 46 if s % 2 else 76, 93e6 if s % 2 else 85e6,
                                    extra_frac=0.1 * (s % 4), interleave_frac=0.1 * (s % 3),
                                    small_frac=0.05 * (s % 5)) for s in seeds]
    _compare(traces, P.variants(capacity=80 * GiB), width)


def test_big_tables_width32():
    """Long runs of equal sizes: the PIN search crosses many words, sorted-set
    shifts span several warp-wide blocks, sBlock groups exceed 32 lanes."""
    traces = [synth.random_trace(100 + s, 3000, 400, sizes=[2 * MiB, 4 * MiB, 6 * MiB, 64 * MiB, 130 * MiB],
                                 p_malloc=0.6) for s in range(2)]
    pols = P.variants(capacity=200 * GiB)
    for p in pols[2:]:
        p["frag_limit_bytes"] = 4 * MiB
    _compare(traces, pols, 32)


def test_c2_width1():
    """BASELINE configs[1] (C2, OPT-1.3B + recompute, 121,968 events), all 8
    variants, through the host executor."""
    ev, _ = synth.config_c2()
    _compare([ev], P.variants(capacity=80 * GiB) + [P.spool64(80 * GiB)], 1)


def test_c3_c4_width1():
    traces = [synth.config_c3(0)[0]]
    _compare(traces, P.variants(capacity=80 * GiB), 1)
    _compare([synth.config_c4(1777)[0]], P.variants(capacity=180 * GiB), 1)


def test_c2_prefix_width32_free_runs():
    """The kernel's window loop with batched frees (Engine::free_run: runs of
    consecutive VMM-path frees unbound at once, sBlock intervals spread over
    the lanes) on the first 3 C2 iterations, all 8 variants, emulated warp."""
    ev, _ = synth.config_c2()
    _compare([ev[:12000]], P.variants(capacity=80 * GiB), 32)


def _lazy_pin_trace(rounds=60):
    """Three 4 MiB blocks, two of them freed and stitched into an 8 MiB
    sBlock, which is then re-bound (S1 sPool hit) and freed `rounds` times
    with no pPool search in between -- every re-bind pushes the lazy-PIN
    stack, 20 rounds in a row fill a 16-entry stack (flush on full) -- and
    every 25th round a 2 MiB request searches the pPool (a flush), some
    while the sBlock is bound (a live pending row)."""
    ev = [("m", 0, 4 * MiB), ("m", 1, 4 * MiB), ("m", 2, 4 * MiB), ("f", 0, 0), ("f", 1, 0),
          ("m", 3, 8 * MiB)]
    for i in range(rounds):
        ev.append(("f", 3, 0))
        ev.append(("m", 3, 8 * MiB))
        if i % 25 == 20:
            ev += [("m", 4, 2 * MiB), ("f", 4, 0)]
        if i % 25 == 22:                      # a search while the sBlock is bound (flush of a live pending row)
            ev += [("m", 5, 6 * MiB), ("f", 5, 0)]
    return pack(ev)


@pytest.mark.parametrize("width", [101, 132])
def test_lazy_pin_stack_fills_tiny_tables(width):
    """Lazy PIN (policy.cuh pin_defer / pin_flush) with a 16-entry sPool, so
    the pending stack fills with stale entries and flushes itself; records
    and statistics equal the oracle's, table maxima within the tiny class."""
    tr = _lazy_pin_trace()
    pols = P.variants(capacity=64 * MiB)
    for p in pols[2:]:
        p["frag_limit_bytes"] = 2 * MiB
    for pol in pols:
        a, s, ovf = E.replay(tr, pol, width)
        ao, so = O.replay(tr, pol)
        assert ovf == 0
        assert np.array_equal(a, ao), (pol, int(np.nonzero(a != ao)[0][0]))
        assert s == so
    # the trace does what it says: the sBlock is re-bound by S1 hits
    recs = O.replay(tr, pols[3])[0]
    states = (recs >> np.uint64(34)) & np.uint64(7)
    kinds = (recs >> np.uint64(32)) & np.uint64(3)
    assert int(((states == 1) & (kinds == 1)).sum()) >= 50
