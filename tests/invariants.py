"""Brute-force re-derivation of every decision and invariant, driven event by
event through the oracle's state dumps (tests only).

The checks are written from the paper's definitions, independently of the
oracle's sorted-set walks:
  * S1 = first exact-size inactive block in pool order (Alg. 1 L2-4, PAPER.md
    L404-411; D5); sBlock inactivity from the chunk sets of the live handles
    (D18).
  * S2 = minimum size > b among eligible inactive pBlocks, ties -> highest
    ordinal (Alg. 1 L6-8; D6, D8); S3 = shortest descending prefix with
    sum >= b (L9-10, L462-466); S4 = all of them, sum < b (L466, L524-527);
    S5 iff the shortfall exceeds capacity (L528).
  * I1-I8, I10, BFC tiling / coalescing /
    best-fit minimality.
"""
from __future__ import annotations

import oracle_lib as O
from tracegen import decode
from tracegen import policies as P

NONE = -1


class Violation(AssertionError):
    pass


def _need(cond, msg):
    if not cond:
        raise Violation(msg)


def _bfc_round(raw):
    return 512 if raw < 512 else (raw + 511) // 512 * 512


class Checker:
    def __init__(self, pol: dict, check_lru: bool = True):
        self.pol = pol
        self.s = O.Stepper(pol)
        self.G = pol["chunk_bytes"]
        self.kind = pol["kind"]
        self.flags = pol["flags"]
        self.prev_C = 0
        self.peaks = dict(active=0, reserved=0, requested=0, active_vmm=0, reserved_vmm=0)
        self.raw_of = {}
        self.n = 0

    # ------------------------------------------------------------ snapshots
    def snap(self):
        s = self.s
        return dict(p=s.pblocks(), sb=s.sblocks(), bfc=s.bfc(), h=s.handles(), c=s.counters())

    @staticmethod
    def chunk_sets(sn):
        pb = {r[0]: r for r in sn["p"]}
        sb = {b["ord"]: b for b in sn["sb"]}
        sets = {}
        for slot, kind, ordv, _bytes, _raw in sn["h"]:
            if kind == 0:
                r = pb[ordv]
                sets[slot] = set(range(r[1], r[1] + r[2]))
            elif kind == 1:
                sets[slot] = {c for lo, n in sb[ordv]["iv"] for c in range(lo, lo + n)}
        return sets

    # --------------------------------------------------------------- checks
    def invariants(self, sn, state):
        G = self.G
        c = sn["c"]
        # I1: pBlocks partition [0, C)
        rng = sorted((r[1], r[2]) for r in sn["p"])
        pos = 0
        for lo, n in rng:
            _need(lo == pos and n > 0, f"I1 pBlock tiling broken at {lo}")
            pos = lo + n
        _need(pos == c["C"], "I1 union != [0, C)")
        # I2: chunk exclusivity among live handles
        sets = self.chunk_sets(sn)
        seen = set()
        for slot, cs in sets.items():
            _need(not (cs & seen), f"I2 chunk shared by two live handles (slot {slot})")
            seen |= cs
        # owner field consistency with the handle chunk sets
        owner_of = {}
        for slot, cs in sets.items():
            for ch in cs:
                owner_of[ch] = slot
        for o, lo, n, owner in sn["p"]:
            exp = owner_of.get(lo, NONE)
            _need(owner == exp, f"pBlock {o} owner {owner} != {exp}")
            _need(all(owner_of.get(ch, NONE) == exp for ch in range(lo, lo + n)),
                  f"pBlock {o} partially owned")
        # I3 + I6: sBlocks
        starts = {lo for lo, _ in rng}
        ends = {lo + n for lo, n in rng}
        for b in sn["sb"]:
            _need(b["size"] == sum(n for _, n in b["iv"]), "I3 size != sum of parts")
            _need(len(b["iv"]) >= 2, "I3 sBlock with < 2 members")
            for lo, n in b["iv"]:
                _need(0 <= lo and lo + n <= c["C"], "I6 interval outside pPool")
                _need(lo in starts and (lo + n) in ends, "I6 interval cuts a pBlock")
        # I4, accounting
        _need(c["active"] <= c["reserved"], "I4 active > reserved")
        _need(c["active"] == sum(h[3] for h in sn["h"]), "active != sum of bound blocks")
        _need(c["requested"] == sum(h[4] for h in sn["h"]), "requested != sum of raw")
        _need(c["active_vmm"] == sum(h[3] for h in sn["h"] if h[1] in (0, 1)), "active_vmm")
        _need(c["reserved_vmm"] == c["C"] * G, "reserved_vmm != C*G")
        # I7 / I8: reserved_vmm grows only, and only in S4
        _need(c["C"] >= self.prev_C, "I7 reserved_vmm decreased")
        if c["C"] != self.prev_C:
            _need(state == 4, f"I8 chunks created outside S4 (state {state})")
        self.prev_C = c["C"]
        # BFC: tiling and coalescing fixpoint per segment
        segs = {}
        for seg, off, size, alloc, pool in sn["bfc"]:
            segs.setdefault(seg, []).append((off, size, alloc))
        for seg, bl in segs.items():
            pos = 0
            for i, (off, size, alloc) in enumerate(bl):
                _need(off == pos and size > 0, f"BFC tiling broken in seg {seg}")
                pos = off + size
                if i and not alloc and not bl[i - 1][2]:
                    _need(False, f"BFC adjacent free blocks in seg {seg}")
        # peaks
        for k in self.peaks:
            self.peaks[k] = max(self.peaks[k], c[k])

    def expect_vmm(self, sn, raw):
        """Brute-force S1..S5 decision from the pre-state."""
        G, pol = self.G, self.pol
        b = -(-raw // G)
        sets = self.chunk_sets(sn)
        owned = set().union(*sets.values()) if sets else set()
        inactive_s = [x for x in sn["sb"]
                      if not any(ch in owned for lo, n in x["iv"] for ch in range(lo, lo + n))]
        inactive_p = [r for r in sn["p"] if r[3] == NONE]
        s1_s = [x for x in inactive_s if x["size"] == b]
        s1_p = [r for r in inactive_p if r[2] == b]
        order = [("p", s1_p), ("s", s1_s)] if self.flags & P.F_S1_PBLOCK_FIRST else [("s", s1_s), ("p", s1_p)]
        for kind, lst in order:
            if lst:
                return dict(state=1, kind=0 if kind == "p" else 1,
                            ord=lst[0][0] if kind == "p" else lst[0]["ord"], b=b)
        rr = self.flags & P.F_REMAINDER_RULE
        elig = [r for r in inactive_p if r[2] * G >= pol["frag_limit_bytes"]]
        big = [r for r in (inactive_p if rr else elig) if r[2] > b]
        if big:
            m = min(r[2] for r in big)
            P_ = max((r for r in big if r[2] == m), key=lambda r: r[0])
            return dict(state=2, P=P_, b=b)
        acc, cb = 0, []
        for r in elig:                      # pool order = descending size
            if acc >= b:
                break
            cb.append(r)
            acc += r[2]
        if acc >= b:
            return dict(state=3, CB=cb, acc=acc, b=b)
        short = b - acc
        if sn["c"]["reserved"] + short * G > pol["capacity_bytes"]:
            return dict(state=5, b=b)
        return dict(state=4, CB=cb, acc=acc, b=b, C=sn["c"]["C"])

    def check_vmm(self, exp, rec, pre, post):
        G = self.G
        f = O.rec_fields(rec)
        _need(f["state"] == exp["state"], f"state {f['state']} != expected {exp['state']}")
        st, b = exp["state"], exp["b"]
        rr = self.flags & P.F_REMAINDER_RULE
        pb = {r[0]: r for r in post["p"]}
        sb = {x["ord"]: x for x in post["sb"]}
        if st == 5:
            _need(f["ord"] == 0xFFFFFFFF, "S5 record")
            return
        if st == 1:
            _need((f["kind"], f["ord"]) == (exp["kind"], exp["ord"]), "S1 picked the wrong block")
        elif st == 2:
            Pb = exp["P"]
            whole = rr and (Pb[2] - b) * G < self.pol["frag_limit_bytes"]
            if whole:
                _need(f["kind"] == 0 and f["ord"] == Pb[0], "S2 whole-block assignment")
            else:
                F = pb[f["ord"]]
                _need(f["kind"] == 0 and (F[1], F[2]) == (Pb[1], b), "S2 split front")
                _need(Pb[0] not in pb, "S2 split parent still in pPool")
                _need(any(r[1] == Pb[1] + b and r[2] == Pb[2] - b for r in post["p"]), "S2 remainder")
                if not self.flags & P.F_NO_COMPANION:
                    comp = [x for x in post["sb"] if x["iv"] == [(Pb[1], b), (Pb[1] + b, Pb[2] - b)]]
                    _need(comp or len(post["sb"]) >= self.pol["spool_max_entries"], "S2 companion missing")
        elif st == 3:
            cb, acc = exp["CB"], exp["acc"]
            iv = [(r[1], r[2]) for r in cb]
            if acc > b:
                last = cb[-1]
                nfront = b - (acc - last[2])
                if not (rr and (last[2] - nfront) * G < self.pol["frag_limit_bytes"]):
                    iv[-1] = (last[1], nfront)
            _need(f["kind"] == 1 and sb[f["ord"]]["iv"] == iv, f"S3 stitch {sb.get(f['ord'])} != {iv}")
        elif st == 4:
            cb, acc = exp["CB"], exp["acc"]
            new = (exp["C"], b - acc)
            if not cb:
                _need(f["kind"] == 0 and (pb[f["ord"]][1], pb[f["ord"]][2]) == new, "S4 direct Alloc")
            else:
                iv = [(r[1], r[2]) for r in cb] + [new]
                _need(f["kind"] == 1 and sb[f["ord"]]["iv"] == iv, "S4 stitch members")
        # I10: bound size == b unless REMAINDER_RULE
        hb = {h[0]: h for h in post["h"]}
        if not rr:
            _need(any(h[3] == b * G for h in hb.values()), "I10 bound size != b")

    def expect_bfc(self, sn, raw, small_path):
        r = _bfc_round(raw)
        exact = self.kind == P.BFC_EXACT
        pool = 0 if exact else (0 if r <= (1 << 20) else 1)
        cands = [(size, seg, off) for seg, off, size, alloc, pl in sn["bfc"]
                 if not alloc and pl == pool and size >= r]
        return min(cands) if cands else None

    # ---------------------------------------------------------------- drive
    def step(self, ev):
        is_free, slot, raw = decode(ev)
        pre = self.snap()
        exp = None
        vmm = False
        if not is_free:
            if self.kind == P.GMLAKE and raw >= self.pol["small_threshold_bytes"]:
                vmm = True
                if self.pol["spool_max_inactive_bytes"] >= (1 << 62):
                    exp = self.expect_vmm(pre, raw)
            else:
                exp = ("bfc", self.expect_bfc(pre, raw, self.kind == P.GMLAKE))
        status, rec = self.s.step(ev)
        post = self.snap()
        f = O.rec_fields(rec)
        if status:
            _need(f["state"] == 5, "terminated without S5 record")
            return False
        if vmm and exp is not None:
            self.check_vmm(exp, rec, pre, post)
        elif exp is not None:
            best = exp[1]
            if best is not None:
                _need(f["state"] == 6 and (f["seg"], f["ord"] * 512) == (best[1], best[2]),
                      f"BFC best fit {best} != record {f}")
            else:
                _need(f["state"] == 7, "BFC should open a new segment")
        self.invariants(post, f["state"] if not is_free else 0)
        self.n += 1
        return True

    def run(self, events):
        for ev in events:
            if not self.step(int(ev)):
                break
        st = self.s.stats()
        _need(st["peak_active_bytes"] == self.peaks["active"], "peak active")
        _need(st["peak_reserved_bytes"] == self.peaks["reserved"], "peak reserved")
        _need(st["peak_requested_bytes"] == self.peaks["requested"], "peak requested")
        _need(st["peak_active_vmm_bytes"] == self.peaks["active_vmm"], "peak active vmm")
        _need(st["peak_reserved_vmm_bytes"] == self.peaks["reserved_vmm"], "peak reserved vmm")
        return st


def theorem_holds(timeline) -> bool:
    """No-new-peak theorem with limit = 1 chunk: the VMM
    reserved bytes after each event equal the running max of VMM active."""
    import numpy as np
    av = timeline[:, 2].astype(np.int64)
    rv = timeline[:, 3].astype(np.int64)
    return bool(np.array_equal(rv, np.maximum.accumulate(av)))
