"""Property-based parity (hypothesis): random traces x random policies
(capacity, fragmentation limit, sPool caps, every flag combination) through
the product engine on the CPU (tests/engine_host.cpp, width 1 and the
emulated 32-lane warp) must equal the oracle record for record. Hypothesis
shrinks any counterexample to a minimal trace."""
import numpy as np
from hypothesis import given, settings, strategies as st, HealthCheck

import engine_lib as E
import oracle_lib as O
from tracegen import SlotAssigner
from tracegen import policies as P

MiB = 1 << 20
SIZES = [1, 512, 513, 300 * 1024, 1536 * 1024, 2 * MiB - 1, 2 * MiB, 3 * MiB, 4 * MiB, 6 * MiB, 10 * MiB,
         14 * MiB, 40 * MiB, 128 * MiB - 1, 128 * MiB, 130 * MiB]


@st.composite
def traces(draw):
    n = draw(st.integers(1, 120))
    sa = SlotAssigner()
    live, nxt = [], 0
    for _ in range(n):
        if live and draw(st.booleans()) and draw(st.booleans()):
            sa.free(live.pop(draw(st.integers(0, len(live) - 1))))
        else:
            sa.malloc(nxt, draw(st.sampled_from(SIZES)))
            live.append(nxt)
            nxt += 1
    if draw(st.booleans()):
        for t in live:
            sa.free(t)
    return np.array(sa.events, dtype=np.uint64)


@st.composite
def policies(draw):
    kind = draw(st.sampled_from([P.GMLAKE, P.GMLAKE, P.GMLAKE, P.BFC_TORCH, P.BFC_EXACT]))
    cap = draw(st.sampled_from([12, 24, 48, 96, 512, 4096])) * MiB
    if kind != P.GMLAKE:
        return P.policy(kind, capacity=cap)
    flags = draw(st.integers(0, 31))
    limit = draw(st.sampled_from([2, 4, 6, 16, 128])) * MiB
    spool = draw(st.sampled_from([1, 2, 3, 8, 4096]))
    byte_cap = draw(st.sampled_from([None, 4 * MiB, 16 * MiB, 64 * MiB]))
    return P.policy(P.GMLAKE, flags, capacity=cap, frag_limit=limit, spool_max_entries=spool,
                    spool_max_inactive_bytes=byte_cap)


def _check(ev, pol, width):
    a, s, ovf = E.replay(ev, pol, width)
    ao, so = O.replay(ev, pol)
    assert ovf == 0
    assert np.array_equal(a, ao), [(i, O.rec_fields(a[i]), O.rec_fields(ao[i])) for i in np.nonzero(a != ao)[0][:3]]
    assert s == so, {k: (s[k], so[k]) for k in so if s[k] != so[k]}


@settings(max_examples=2000, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(traces(), policies())
def test_engine_width1_equals_oracle(ev, pol):
    _check(ev, pol, 1)


@settings(max_examples=200, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(traces(), policies())
def test_engine_warp_emulation_equals_oracle(ev, pol):
    _check(ev, pol, 32)
