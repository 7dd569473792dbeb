"""Brute-force re-derivation of every decision and invariant, driven event by
event through the oracle's state dumps (tests only).

The checks are written from the paper's definitions, independently of the
oracle's sorted-set walks, and they are TWO-WAY: a step that terminates the
trace is checked against the brute-force expectation too (an OOM is right iff
the definitions say so).
  * S1 = first exact-size inactive block in pool order (Alg. 1 L2-4, PAPER.md
    L404-411; D5); sBlock inactivity from the chunk sets of the live handles
    (D18).
  * S2 = minimum size > b among eligible inactive pBlocks, ties -> highest
    ordinal (Alg. 1 L6-8; D6, D8); S3 = shortest descending prefix with
    sum >= b (L9-10, L462-466); S4 = all of them, sum < b (L466, L524-527);
    S5 iff the shortfall exceeds capacity once the small path has returned
    its fully free segments (L528, D16); under D8' (LIMIT_GATES_REQUEST) a
    request below the fragmentation limit takes the small path (L571, L322).
  * StitchFree (D17): the set of sBlocks a
    malloc removes is re-derived as a set: the byte cap at malloc entry
    (least recently used inactive first until the inactive bytes fit), the
    SPLIT_INVALIDATES variant (every sBlock over the split parent, SPEC.md
    L324), and the count cap at each Stitch (least recently used inactive
    sBlock not created during this malloc; a companion with no room is
    skipped). LRU key = touch at creation or S1 reuse.
  * BFC (D21-D23): best fit = min (size, address) by a
    linear scan, the split decision, the new segment's size, and the OOM path:
    release every fully free segment, retry once, OOM iff it still does not
    fit.
  * I1-I8, I10, BFC tiling / coalescing.
"""
from __future__ import annotations

import oracle_lib as O
from tracegen import decode
from tracegen import policies as P

NONE = -1
MiB = 1 << 20

# D21 (PyTorch CUDACachingAllocator constants, pinned by the hand goldens in
# tests/golden/bfc_d21.json and by I13 on the GPU)
K_MIN_BLOCK, K_SMALL_SIZE, K_SMALL_BUFFER = 512, 1 * MiB, 2 * MiB
K_MIN_LARGE_ALLOC, K_LARGE_BUFFER, K_ROUND_LARGE = 10 * MiB, 20 * MiB, 2 * MiB

# vmm_calls index (D26)
V_RESERVE, V_CREATE, V_MAP, V_ACCESS, V_UNMAP, V_ADDR_FREE = range(6)


class Violation(AssertionError):
    pass


def _need(cond, msg):
    if not cond:
        raise Violation(msg)


def _bfc_round(raw):
    return K_MIN_BLOCK if raw < K_MIN_BLOCK else (raw + K_MIN_BLOCK - 1) // K_MIN_BLOCK * K_MIN_BLOCK


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
        self.n_oom = 0
        self.n_evict_checked = 0
        self.n_release_checked = 0

    # ------------------------------------------------------------ snapshots
    def snap(self):
        s = self.s
        return dict(p=s.pblocks(), sb=s.sblocks(), bfc=s.bfc(), h=s.handles(), c=s.counters(),
                    st=s.stats())

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

    @classmethod
    def owned(cls, sn):
        sets = cls.chunk_sets(sn)
        return set().union(*sets.values()) if sets else set()

    @staticmethod
    def s_inactive(x, owned):
        return not any(ch in owned for lo, n in x["iv"] for ch in range(lo, lo + n))

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
        # pool order (D4): size descending, ordinal ascending
        keys = [(-r[2], r[0]) for r in sn["p"]]
        _need(keys == sorted(keys), "pPool not in (size desc, ordinal asc) order")
        skeys = [(-b["size"], b["ord"]) for b in sn["sb"]]
        _need(skeys == sorted(skeys), "sPool not in (size desc, ordinal asc) order")
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
        segs = {}
        for seg, off, size, alloc, pool in sn["bfc"]:
            segs.setdefault(seg, []).append((off, size, alloc))
        _need(c["reserved"] == c["C"] * G + sum(sz for bl in segs.values() for _, sz, _ in bl),
              "reserved != chunks + BFC segments (D20)")
        # I7 / I8: reserved_vmm grows only, and only in S4
        _need(c["C"] >= self.prev_C, "I7 reserved_vmm decreased")
        if c["C"] != self.prev_C:
            _need(state == 4, f"I8 chunks created outside S4 (state {state})")
        self.prev_C = c["C"]
        # BFC: tiling and coalescing fixpoint per segment
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

    # ------------------------------------------------------- VMM decisions
    def byte_cap_victims(self, sn):
        """D17(ii) at VMM-path malloc entry: while the inactive sBlocks hold
        more than spool_max_inactive_bytes, the least recently used inactive
        one goes."""
        G, cap = self.G, self.pol["spool_max_inactive_bytes"]
        owned = self.owned(sn)
        inact = sorted((x for x in sn["sb"] if self.s_inactive(x, owned)), key=lambda x: x["last_use"])
        tot = sum(x["size"] * G for x in inact)
        out = []
        for x in inact:
            if tot <= cap:
                break
            out.append(x["ord"])
            tot -= x["size"] * G
        return out

    def expect_vmm(self, sn, raw):
        """Brute-force S1..S5 decision from the pre-state."""
        G, pol = self.G, self.pol
        b = -(-raw // G)
        owned = self.owned(sn)
        inactive_s = [x for x in sn["sb"] if self.s_inactive(x, owned)]
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
        release = []
        res = sn["c"]["reserved"]
        if res + short * G > pol["capacity_bytes"]:
            # D16: the small path returns its fully free segments first
            release = self.free_segments(sn)
            res -= sum(sz for seg, off, sz, alloc, pl in sn["bfc"] if seg in release)
        if res + short * G > pol["capacity_bytes"]:
            return dict(state=5, b=b, release=release)
        return dict(state=4, CB=cb, acc=acc, b=b, C=sn["c"]["C"], release=release)

    @staticmethod
    def free_segments(sn):
        """BFC segments that are one free block (PyTorch's releasable cache)."""
        segs = {}
        for seg, off, size, alloc, pl in sn["bfc"]:
            segs.setdefault(seg, []).append((size, alloc))
        return sorted(s for s, bl in segs.items() if len(bl) == 1 and not bl[0][1])

    def expect_spool_ops(self, exp, sn, owned):
        """The sPool transition of one VMM malloc after the byte-cap phase:
        -> (victim ordinals in order, expected new sBlocks as member interval
        lists, companion interval lists skipped for lack of room)."""
        G, rr = self.G, self.flags & P.F_REMAINDER_RULE
        cap = self.pol["spool_max_entries"]
        pool = [dict(ord=x["ord"], last_use=x["last_use"], iv=x["iv"], inactive=self.s_inactive(x, owned),
                     new=False) for x in sn["sb"]]
        victims, created, skipped = [], [], []

        def split(Pb):
            if self.flags & P.F_SPLIT_INVALIDATES:     # every sBlock over the parent
                lo, n = Pb[1], Pb[2]
                for x in list(pool):
                    if any(a < lo + n and lo < a + m for a, m in x["iv"]):
                        pool.remove(x)
                        victims.append(x["ord"])

        def stitch(iv, companion):
            while len(pool) >= cap:
                cands = [x for x in pool if x["inactive"] and not x["new"]]
                if not cands:
                    break
                v = min(cands, key=lambda x: x["last_use"])
                pool.remove(v)
                victims.append(v["ord"])
            if companion and len(pool) >= cap:
                skipped.append(iv)
                return
            pool.append(dict(ord=None, last_use=None, iv=iv, inactive=companion, new=True))
            created.append((iv, companion))

        st, b = exp["state"], exp["b"]
        nocomp = self.flags & P.F_NO_COMPANION
        if st == 2:
            Pb = exp["P"]
            if not (rr and (Pb[2] - b) * G < self.pol["frag_limit_bytes"]):
                split(Pb)
                if not nocomp:
                    stitch([(Pb[1], b), (Pb[1] + b, Pb[2] - b)], True)
        elif st == 3:
            cb, acc = exp["CB"], exp["acc"]
            iv = [(r[1], r[2]) for r in cb]
            if acc > b:
                last = cb[-1]
                nf = b - (acc - last[2])
                if not (rr and (last[2] - nf) * G < self.pol["frag_limit_bytes"]):
                    split(last)
                    if not nocomp:
                        stitch([(last[1], nf), (last[1] + nf, last[2] - nf)], True)
                    iv[-1] = (last[1], nf)
            stitch(iv, False)
        elif st == 4 and exp["CB"]:
            stitch([(r[1], r[2]) for r in exp["CB"]] + [(exp["C"], b - exp["acc"])], False)
        return victims, created, skipped

    def check_vmm(self, exp, rec, pre, post):
        G = self.G
        f = O.rec_fields(rec)
        _need(f["state"] == exp["state"], f"state {f['state']} != expected {exp['state']}")
        st, b = exp["state"], exp["b"]
        pre_segs, post_segs = {x[0] for x in pre["bfc"]}, {x[0] for x in post["bfc"]}
        _need(pre_segs - post_segs == set(exp.get("release", [])),
              f"small-path segments released {sorted(pre_segs - post_segs)} != {exp.get('release', [])} (D16)")
        if exp.get("release"):
            self.n_release_checked += 1
        rr = self.flags & P.F_REMAINDER_RULE
        pb = {r[0]: r for r in post["p"]}
        sb = {x["ord"]: x for x in post["sb"]}
        if st == 5:
            _need(f["ord"] == 0xFFFFFFFF, "S5 record")
            return
        if st == 1:
            _need((f["kind"], f["ord"]) == (exp["kind"], exp["ord"]), "S1 picked the wrong block")
            if f["kind"] == 1:     # LRU key = the touch of this reuse (D17)
                _need(sb[f["ord"]]["last_use"] == max(x["last_use"] for x in post["sb"]),
                      "S1 sBlock reuse did not refresh its LRU key")
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

    def check_spool(self, pre, post, victims, created, skipped, stopped):
        n_comp = sum(1 for _, c in created if c)
        created = [iv for iv, _ in created]
        """The sBlocks a malloc removed and created, as sets (D17, SPEC.md
        L324), and the counters that follow them (D26)."""
        pre_o = {x["ord"] for x in pre["sb"]}
        post_o = {x["ord"] for x in post["sb"]}
        gone = pre_o - post_o
        _need(gone == set(victims), f"evicted {sorted(gone)} != expected {sorted(victims)}")
        if stopped:
            return
        new = [x for x in post["sb"] if x["ord"] not in pre_o]
        _need(sorted(tuple(map(tuple, x["iv"])) for x in new) == sorted(tuple(v) for v in created),
              f"created sBlocks {[x['iv'] for x in new]} != expected {created}")
        if new:   # a new sBlock's LRU key is a fresh touch (creation)
            old = max((x["last_use"] for x in pre["sb"]), default=0)
            _need(all(x["last_use"] > old for x in new), "new sBlock LRU key not fresh")
        d = {k: post["st"][k] - pre["st"][k] for k in ("n_evict", "n_stitch", "n_companion")}
        _need(d["n_evict"] == len(victims), "n_evict delta")
        _need(d["n_stitch"] == len(created), "n_stitch delta")
        _need(d["n_companion"] == n_comp, "n_companion delta")
        dv = [post["st"]["vmm_calls"][i] - pre["st"]["vmm_calls"][i] for i in range(7)]
        _need(dv[V_UNMAP] >= len(victims) and dv[V_ADDR_FREE] >= len(victims), "StitchFree calls (D26)")
        if victims or created or skipped:
            self.n_evict_checked += bool(victims)

    # ------------------------------------------------------------------ BFC
    def expect_bfc(self, sn, raw):
        """Best fit, split and segment decisions of BFC (V0, V1, GMLake's
        small path) from the pre-state: PAPER.md L116-125, D21-D23."""
        r = _bfc_round(raw)
        exact = self.kind == P.BFC_EXACT
        pool = 0 if exact else (0 if r <= K_SMALL_SIZE else 1)
        cands = [(size, seg, off) for seg, off, size, alloc, pl in sn["bfc"]
                 if not alloc and pl == pool and size >= r]
        best = min(cands) if cands else None
        out = dict(r=r, pool=pool, best=best, exact=exact)
        if best is None:
            ss = r if exact else (K_SMALL_BUFFER if r <= K_SMALL_SIZE else
                                  K_LARGE_BUFFER if r < K_MIN_LARGE_ALLOC else
                                  -(-r // K_ROUND_LARGE) * K_ROUND_LARGE)
            out["ss"] = ss
            res, cap = sn["c"]["reserved"], self.pol["capacity_bytes"]
            free_segs = self.free_segments(sn)
            freed = sum(sz for seg, off, sz, alloc, pl in sn["bfc"] if seg in free_segs)
            if res + ss <= cap:
                out["release"] = []
            else:
                out["release"] = free_segs
                out["oom"] = res - freed + ss > cap
            size = ss
        else:
            size = best[0]
        rem = size - r
        out["split"] = rem >= K_MIN_BLOCK if (exact or pool == 0) else rem > K_SMALL_SIZE
        out["alloc_size"] = r if out["split"] else size
        return out

    def check_bfc(self, e, f, pre, post, stopped):
        pre_segs = {b[0] for b in pre["bfc"]}
        post_segs = {b[0] for b in post["bfc"]}
        if e["best"] is None and e["release"]:
            _need(pre_segs - post_segs == set(e["release"]),
                  f"released segments {sorted(pre_segs - post_segs)} != {e['release']}")
            self.n_release_checked += 1
        elif not stopped:
            _need(pre_segs <= post_segs, "a segment was released without an OOM retry")
        if e.get("oom"):
            _need(stopped and f["state"] == 5, "BFC should report OOM after release-and-retry")
            return
        _need(not stopped, f"BFC reported OOM where a fit exists: {e}")
        if e["best"] is not None:
            _need(f["state"] == 6 and (f["seg"], f["ord"] * 512) == (e["best"][1], e["best"][2]),
                  f"BFC best fit {e['best']} != record {f}")
        else:
            _need(f["state"] == 7, "BFC should open a new segment")
            segsz = sum(b[2] for b in post["bfc"] if b[0] == f["seg"])
            _need(segsz == e["ss"], f"new segment {segsz} != {e['ss']} (D21)")
        blk = [b for b in post["bfc"] if b[0] == f["seg"] and b[1] == f["ord"] * 512]
        _need(len(blk) == 1 and blk[0][3] == 1, "allocated BFC block not found")
        _need(blk[0][2] == e["alloc_size"], f"BFC allocated {blk[0][2]} != {e['alloc_size']} (split rule)")

    # ---------------------------------------------------------------- drive
    def step(self, ev):
        is_free, slot, raw = decode(ev)
        pre = self.snap()
        exp = None
        kind = None
        if not is_free:
            gate = self.flags & P.F_LIMIT_GATES_REQUEST and raw < self.pol["frag_limit_bytes"]   # D8'
            if self.kind == P.GMLAKE and raw >= self.pol["small_threshold_bytes"] and not gate:
                kind = "vmm"
                v0 = self.byte_cap_victims(pre)
                pre_d = dict(pre, sb=[x for x in pre["sb"] if x["ord"] not in v0])
                exp = self.expect_vmm(pre_d, raw)
                ops = ([], [], []) if exp["state"] == 5 else \
                    self.expect_spool_ops(exp, pre_d, self.owned(pre_d))
                victims = v0 + ops[0]
            else:
                kind = "bfc"
                exp = self.expect_bfc(pre, raw)
        status, rec = self.s.step(ev)
        post = self.snap()
        f = O.rec_fields(rec)
        stopped = bool(status)
        if stopped:
            _need(f["state"] == 5, "terminated without S5 record")
            self.n_oom += 1
        if kind == "vmm":
            self.check_vmm(exp, rec, pre, post)
            self.check_spool(pre, post, victims, ops[1], ops[2], stopped)
        elif kind == "bfc":
            self.check_bfc(exp, f, pre, post, stopped)
        if stopped:
            return False
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
