"""The decomposition the split and path units rest on, checked
on the oracle alone (no GPU): a GMLake unit's VMM path and small path share
only the capacity (requests below the gate take PyTorch's
splitting method; L524-528: S4/S5 against the capacity), so while no
capacity check fails, replaying the two sub-traces separately gives the
interleaved replay's records event by event, its counters as sums, its
reserved peak as the sum of the finals, and its active peak as the maximum
of the two paths' active bytes summed in event order. When the paths'
reserved bytes together exceed the capacity the decomposition may break,
which is why the kernels hand such units back to the single-warp replay."""
import numpy as np
import pytest

import oracle_lib as O
from tracegen import synth
from tracegen import policies as P

GiB = 1 << 30
MiB = 1 << 20


def _gate(p):
    g = p["small_threshold_bytes"]
    if p["flags"] & P.F_LIMIT_GATES_REQUEST and p["frag_limit_bytes"] > g:
        g = p["frag_limit_bytes"]
    return g


def _paths(ev, gate):
    """event indices of the VMM path and of the small path (a free follows its malloc)"""
    ev = np.asarray(ev, dtype=np.uint64)
    big, last = np.zeros(len(ev), bool), {}
    for i, e in enumerate(ev.tolist()):
        slot = (e >> 40) & 0x7FFFFF
        if e >> 63:
            big[i] = last.pop(slot)
        else:
            big[i] = (e & ((1 << 40) - 1)) >= gate
            last[slot] = big[i]
    return np.nonzero(big)[0], np.nonzero(~big)[0]


def _merge(ev, pol):
    """(records, stats) of the unit rebuilt from its two paths' oracle replays"""
    ev = np.asarray(ev, dtype=np.uint64)
    iv, is_ = _paths(ev, _gate(pol))
    av, sv, tv = O.replay(ev[iv], pol, timeline=True)
    as_, ss, ts = O.replay(ev[is_], pol, timeline=True)
    rec = np.zeros(len(ev), dtype=np.uint64)
    rec[iv], rec[is_] = av, as_
    # active bytes after every event: each path's value after its latest event
    act_v = np.zeros(len(ev), dtype=np.int64)
    act_s = np.zeros(len(ev), dtype=np.int64)
    act_v[iv], act_s[is_] = tv[:, 0].astype(np.int64), ts[:, 0].astype(np.int64)
    own_v = np.zeros(len(ev), bool)
    own_v[iv] = True
    idx_v = np.maximum.accumulate(np.where(own_v, np.arange(len(ev)), -1))
    idx_s = np.maximum.accumulate(np.where(~own_v, np.arange(len(ev)), -1))
    tot = np.where(idx_v >= 0, act_v[np.maximum(idx_v, 0)], 0) + np.where(idx_s >= 0, act_s[np.maximum(idx_s, 0)], 0)
    st = dict(sv)
    st["peak_active_bytes"] = int(tot.max()) if len(ev) else 0
    st["peak_reserved_bytes"] = sv["final_reserved_bytes"] + ss["final_reserved_bytes"]
    st["final_active_bytes"] = sv["final_active_bytes"] + ss["final_active_bytes"]
    st["final_reserved_bytes"] = sv["final_reserved_bytes"] + ss["final_reserved_bytes"]
    st["n_events"] = st["n_events_done"] = len(ev)
    st["state_count"] = sv["state_count"][:5] + ss["state_count"][5:]
    for k in ("n_seg_alloc", "n_seg_release", "max_bfc_blocks"):
        st[k] = ss[k]
    return rec, st, sv, ss


@pytest.mark.parametrize("v", [2, 3, 4, 5, 6, 7])
def test_two_paths_rebuild_the_interleaved_replay(v):
    tr = synth.config_c3(1)[0]
    pol = P.variants(capacity=80 * GiB)[v]
    ao, so = O.replay(tr, pol)
    rec, st, sv, ss = _merge(tr, pol)
    assert sv["status"] == 0 and ss["status"] == 0
    assert sv["final_reserved_bytes"] + ss["final_reserved_bytes"] <= pol["capacity_bytes"]
    assert np.array_equal(rec, ao)
    for k in ("peak_active_bytes", "peak_reserved_bytes", "final_active_bytes", "final_reserved_bytes",
              "peak_active_vmm_bytes", "peak_reserved_vmm_bytes", "state_count", "n_split", "n_stitch",
              "n_companion", "n_alloc", "n_evict", "n_seg_alloc", "n_seg_release", "vmm_calls", "max_pblocks",
              "max_sblocks", "max_bfc_blocks"):
        assert st[k] == so[k], (k, st[k], so[k])
    # the ledger's figures come from the event stream alone
    assert so["peak_requested_bytes"] == O.replay(tr, P.variants(capacity=80 * GiB)[0])[1]["peak_requested_bytes"]


def test_capacity_sum_breaks_the_decomposition():
    """Each path fits the capacity alone, their sum does not: the interleaved
    replay differs from the rebuilt one (an OOM, or a BFC release changing
    later decisions) -- the case the kernels re-run single-warp."""
    tr = synth.config_c3(0)[0]
    big = P.variants(capacity=80 * GiB)[3]
    _, so = O.replay(tr, big)
    rv = so["peak_reserved_vmm_bytes"]
    rs = so["peak_reserved_bytes"] - rv
    cap = max(rv, rs) + min(rv, rs) // 2
    pol = dict(big, capacity_bytes=cap, spool_max_inactive_bytes=cap)
    ao, so2 = O.replay(tr, pol)
    rec, st, sv, ss = _merge(tr, pol)
    assert sv["status"] == 0 and ss["status"] == 0                  # each path alone completes
    assert sv["final_reserved_bytes"] + ss["final_reserved_bytes"] > cap
    assert so2["status"] != 0 or not np.array_equal(rec, ao) or st["peak_reserved_bytes"] != so2["peak_reserved_bytes"]
