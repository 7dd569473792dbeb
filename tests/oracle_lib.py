"""ctypes binding of the CPU oracle (oracle/libgml_oracle.so) for tests and
the bench's cpu_baseline leg. Test infrastructure: never imported by the
product package."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "oracle" / "gml_oracle.cpp"
LIB = ROOT / "oracle" / "libgml_oracle.so"


def build(force: bool = False) -> Path:
    if force or not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        tmp = LIB.with_suffix(f".{os.getpid()}.tmp")
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", str(SRC), "-o", str(tmp)])
        os.replace(tmp, LIB)
    return LIB


class Policy(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("flags", C.c_uint32), ("capacity_bytes", C.c_uint64),
                ("chunk_bytes", C.c_uint64), ("small_threshold_bytes", C.c_uint64),
                ("frag_limit_bytes", C.c_uint64), ("spool_max_entries", C.c_uint32),
                ("_pad", C.c_uint32), ("spool_max_inactive_bytes", C.c_uint64)]


class Stats(C.Structure):
    _fields_ = [("peak_active_bytes", C.c_uint64), ("peak_reserved_bytes", C.c_uint64),
                ("peak_requested_bytes", C.c_uint64), ("peak_active_vmm_bytes", C.c_uint64),
                ("peak_reserved_vmm_bytes", C.c_uint64), ("final_active_bytes", C.c_uint64),
                ("final_reserved_bytes", C.c_uint64), ("n_events", C.c_uint64),
                ("n_events_done", C.c_uint64), ("oom_event", C.c_int64), ("status", C.c_uint32),
                ("_p", C.c_uint32), ("state_count", C.c_uint64 * 7), ("n_split", C.c_uint64),
                ("n_stitch", C.c_uint64), ("n_companion", C.c_uint64), ("n_alloc", C.c_uint64),
                ("n_evict", C.c_uint64), ("n_seg_alloc", C.c_uint64), ("n_seg_release", C.c_uint64),
                ("vmm_calls", C.c_uint64 * 7), ("max_pblocks", C.c_uint32), ("max_sblocks", C.c_uint32),
                ("max_live_handles", C.c_uint32), ("max_bfc_blocks", C.c_uint32)]

    def to_dict(self) -> dict:
        d = {}
        for name, _ in self._fields_:
            if name.startswith("_"):
                continue
            v = getattr(self, name)
            d[name] = list(v) if hasattr(v, "__len__") else int(v)
        return d


_lib = None


def lib():
    global _lib
    if _lib is None:
        # GML_ORACLE_LIB: a prebuilt oracle (tools/oracle_mutants.py points it
        # at deliberately broken copies to check that the pins kill them)
        alt = os.environ.get("GML_ORACLE_LIB")
        L = C.CDLL(alt if alt else str(build()))
        L.gmo_create.restype = C.c_void_p
        L.gmo_create.argtypes = [C.POINTER(Policy)]
        L.gmo_destroy.argtypes = [C.c_void_p]
        L.gmo_step.restype = C.c_uint32
        L.gmo_step.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)]
        L.gmo_get_stats.argtypes = [C.c_void_p, C.POINTER(Stats)]
        for fn in ("gmo_dump_pblocks", "gmo_dump_sblocks", "gmo_dump_bfc", "gmo_dump_handles"):
            getattr(L, fn).restype = C.c_uint64
            getattr(L, fn).argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.c_uint64]
        L.gmo_counters.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
        L.gmo_replay.restype = C.c_uint32
        L.gmo_replay.argtypes = [C.POINTER(C.c_uint64), C.c_uint64, C.POINTER(Policy),
                                 C.POINTER(C.c_uint64), C.POINTER(Stats), C.POINTER(C.c_uint64)]
        L.gmo_sizeof_stats.restype = C.c_uint64
        L.gmo_sizeof_policy.restype = C.c_uint64
        assert L.gmo_sizeof_stats() == C.sizeof(Stats) == 272
        assert L.gmo_sizeof_policy() == C.sizeof(Policy) == 56
        _lib = L
    return _lib


def to_policy(d: dict) -> Policy:
    p = Policy()
    for k, v in d.items():
        setattr(p, k, v)
    return p


def _u64p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def replay(events: np.ndarray, pol: dict, timeline: bool = False):
    """-> (assignments u64[n], stats dict[, timeline u64[n,4]])"""
    ev = np.ascontiguousarray(events, dtype=np.uint64)
    n = len(ev)
    asg = np.zeros(max(n, 1), dtype=np.uint64)
    tl = np.zeros((max(n, 1), 4), dtype=np.uint64) if timeline else None
    st = Stats()
    p = to_policy(pol)
    lib().gmo_replay(_u64p(ev), n, C.byref(p), _u64p(asg), C.byref(st),
                     _u64p(tl) if timeline else None)
    out = (asg[:n], st.to_dict())
    if timeline:
        out = out + (tl[:n],)
    return out


class Stepper:
    """Event-by-event driver with state dumps (invariant tests)."""

    def __init__(self, pol: dict):
        self._p = to_policy(pol)
        self.h = lib().gmo_create(C.byref(self._p))

    def __del__(self):
        if getattr(self, "h", None):
            lib().gmo_destroy(self.h)
            self.h = None

    def step(self, ev: int) -> tuple[int, int]:
        a = C.c_uint64(0)
        status = lib().gmo_step(self.h, int(ev), C.byref(a))
        return status, a.value

    def stats(self) -> dict:
        st = Stats()
        lib().gmo_get_stats(self.h, C.byref(st))
        return st.to_dict()

    def _dump(self, fn, width):
        n = getattr(lib(), fn)(self.h, None, 0)
        buf = np.zeros(max(n * width, 1), dtype=np.int64)
        getattr(lib(), fn)(self.h, buf.ctypes.data_as(C.POINTER(C.c_int64)), n * width)
        return buf[: n * width].reshape(n, width) if width else buf

    def pblocks(self):
        """pool order rows (ord, lo, n, owner)"""
        return [tuple(int(x) for x in r) for r in self._dump("gmo_dump_pblocks", 4)]

    def sblocks(self):
        """pool order: dicts {ord, size, last_use, iv: [(lo, n)]}"""
        n = lib().gmo_dump_sblocks(self.h, None, 0)
        buf = np.zeros(max(n, 1), dtype=np.int64)
        lib().gmo_dump_sblocks(self.h, buf.ctypes.data_as(C.POINTER(C.c_int64)), n)
        out, k = [], 0
        while k < n:
            o, sz, lu, niv = (int(x) for x in buf[k:k + 4])
            k += 4
            iv = [(int(buf[k + 2 * j]), int(buf[k + 2 * j + 1])) for j in range(niv)]
            k += 2 * niv
            out.append(dict(ord=o, size=sz, last_use=lu, iv=iv))
        return out

    def bfc(self):
        """address order rows (seg, off, size, allocated, pool)"""
        return [tuple(int(x) for x in r) for r in self._dump("gmo_dump_bfc", 5)]

    def handles(self):
        """rows (slot, kind, ord_or_seg, bytes, raw)"""
        return [tuple(int(x) for x in r) for r in self._dump("gmo_dump_handles", 5)]

    def counters(self) -> dict:
        buf = (C.c_uint64 * 7)()
        lib().gmo_counters(self.h, buf)
        keys = ["active", "requested", "reserved", "active_vmm", "reserved_vmm", "C", "T"]
        return dict(zip(keys, [int(x) for x in buf]))


def stats_bytes(d: dict) -> bytes:
    """Stats dict -> the 272-byte record (the gml_stats_t layout)."""
    s = Stats()
    for k, v in d.items():
        if isinstance(v, list):
            getattr(s, k)[:] = v
        else:
            setattr(s, k, v)
    return bytes(s)


# assignment-record decoding
def rec_fields(r: int) -> dict:
    r = int(r)
    return dict(ord=r & 0xFFFFFFFF, kind=(r >> 32) & 3, state=(r >> 34) & 7, seg=r >> 40)
