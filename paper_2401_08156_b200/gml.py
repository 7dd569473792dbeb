"""Thin ctypes binding of libgml.so (include/gml.h): argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; there is no
Python or CPU fallback. Importing this module fails loudly when the library
is missing (build it with `python -c "import __graft_entry__ as g; g.build()"`).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("GML_LIB", _HERE / "libgml.so"))

GML_OK, GML_ERR_INVALID, GML_ERR_OOM, GML_ERR_CUDA, GML_ERR_TABLE_OVERFLOW, GML_ERR_UNSUPPORTED = range(6)
GML_POLICY_BFC_TORCH, GML_POLICY_BFC_EXACT, GML_POLICY_GMLAKE = 0, 1, 2


class GmlError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: {status_string(code)} ({code})")
        self.code = code


class gml_policy(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("flags", C.c_uint32), ("capacity_bytes", C.c_uint64),
                ("chunk_bytes", C.c_uint64), ("small_threshold_bytes", C.c_uint64),
                ("frag_limit_bytes", C.c_uint64), ("spool_max_entries", C.c_uint32),
                ("_pad", C.c_uint32), ("spool_max_inactive_bytes", C.c_uint64)]


class gml_stats_t(C.Structure):
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


class gml_replay_caps(C.Structure):
    _fields_ = [("pblocks", C.c_uint32), ("sblocks", C.c_uint32), ("intervals", C.c_uint32),
                ("bfc_blocks", C.c_uint32)]


class gml_trace_batch(C.Structure):
    _fields_ = [("events", C.c_void_p), ("trace_offsets", C.c_void_p), ("n_traces", C.c_uint32),
                ("n_policies", C.c_uint32), ("policies", C.POINTER(gml_policy)),
                ("assignments", C.c_void_p), ("stats", C.c_void_p), ("stream", C.c_void_p),
                ("caps", C.POINTER(gml_replay_caps)), ("timeline", C.c_void_p)]


STATS_DTYPE = np.dtype([(n, np.uint64 if t in (C.c_uint64,) else np.int64 if t is C.c_int64 else np.uint32)
                        if not hasattr(t, "_length_") else (n, np.uint64, (t._length_,))
                        for n, t in gml_stats_t._fields_])
assert STATS_DTYPE.itemsize == 272

_lib = None

# (name, restype, argtypes): every entry point of include/gml.h
SIGNATURES = [
    ("gml_trace_validate", C.c_int, [C.POINTER(C.c_uint64), C.c_uint64, C.POINTER(C.c_uint32)]),
    ("gml_replay", C.c_int, [C.POINTER(gml_trace_batch)]),
    ("gml_last_launch_count", C.c_uint32, []),
    ("gml_last_kernel_ms", C.c_float, []),
    ("gml_last_split_count", C.c_uint32, [C.POINTER(C.c_uint32)]),
    ("gml_utilization", C.c_double, [C.POINTER(gml_stats_t)]),
    ("gml_fragmentation", C.c_double, [C.POINTER(gml_stats_t)]),
    ("gml_create", C.c_int, [C.c_int, C.POINTER(gml_policy), C.POINTER(C.c_void_p)]),
    ("gml_malloc", C.c_int, [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    ("gml_free", C.c_int, [C.c_void_p, C.c_void_p]),
    ("gml_set_stream", C.c_int, [C.c_void_p, C.c_void_p]),
    ("gml_live_trace", C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.c_uint64, C.POINTER(C.c_uint64),
                                 C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    ("gml_cudamalloc_trace", C.c_int, [C.c_int, C.POINTER(C.c_uint64), C.c_uint64, C.POINTER(C.c_uint64),
                                       C.POINTER(C.c_uint64)]),
    ("gml_stats", C.c_int, [C.c_void_p, C.POINTER(gml_stats_t)]),
    ("gml_driver_calls", C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
    ("gml_destroy", C.c_int, [C.c_void_p]),
    ("gml_stream_copy", C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p,
                                  C.POINTER(C.c_float)]),
    ("gml_status_string", C.c_char_p, [C.c_int]),
    ("gml_torch_malloc", C.c_void_p, [C.c_ssize_t, C.c_int, C.c_void_p]),
    ("gml_torch_free", None, [C.c_void_p, C.c_ssize_t, C.c_int, C.c_void_p]),
    ("gml_torch_configure", C.c_int, [C.POINTER(gml_policy)]),
    ("gml_torch_stats", C.c_int, [C.c_int, C.POINTER(gml_stats_t)]),
    ("gml_vmm_profile", C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_int, C.POINTER(C.c_double)]),
]


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"libgml.so not built at {LIB_PATH}; run __graft_entry__.build()")
        L = C.CDLL(str(LIB_PATH))
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def status_string(code: int) -> str:
    return lib().gml_status_string(int(code)).decode()


def _check(code: int, what: str):
    if code != GML_OK:
        raise GmlError(code, what)


def to_policy(d: dict) -> gml_policy:
    p = gml_policy()
    for k, v in d.items():
        setattr(p, k, int(v))
    return p


def policy_array(pols) -> C.Array:
    arr = (gml_policy * len(pols))()
    for i, d in enumerate(pols):
        arr[i] = to_policy(d)
    return arr


def gml_trace_validate(events: np.ndarray) -> int:
    ev = np.ascontiguousarray(events, dtype=np.uint64)
    ms = C.c_uint32(0)
    rc = lib().gml_trace_validate(ev.ctypes.data_as(C.POINTER(C.c_uint64)), len(ev), C.byref(ms))
    if rc != GML_OK:
        raise GmlError(rc, f"gml_trace_validate (bad event {ms.value})")
    return ms.value


def gml_replay(events, trace_offsets, policies, assignments=None, stats=None, stream=None,
               caps: np.ndarray | None = None, timeline=None):
    """Replay on the GPU. `events`, `trace_offsets`, `assignments` and `stats`
    are CUDA tensors (int64 / uint8 views of the packed layouts of gml.h);
    `policies` a list of policy dicts; `caps` an optional uint32 [T*P, 4]
    numpy array of table hints, updated in place; `timeline` an optional
    int64 CUDA tensor [P, total, 2] for (active, reserved) after each event.
    Returns the stats tensor."""
    import torch
    n_traces = trace_offsets.numel() - 1
    n_pol = len(policies)
    if stats is None:
        stats = torch.empty((n_traces * n_pol * 272,), dtype=torch.uint8, device=events.device)
    pols = policy_array(policies)
    b = gml_trace_batch()
    b.events = events.data_ptr()
    b.trace_offsets = trace_offsets.data_ptr()
    b.n_traces = n_traces
    b.n_policies = n_pol
    b.policies = pols
    b.assignments = assignments.data_ptr() if assignments is not None else None
    b.stats = stats.data_ptr()
    b.stream = stream.cuda_stream if stream is not None else torch.cuda.current_stream(events.device).cuda_stream
    if caps is not None:
        assert caps.dtype == np.uint32 and caps.shape == (n_traces * n_pol, 4) and caps.flags.c_contiguous
        b.caps = caps.ctypes.data_as(C.POINTER(gml_replay_caps))
    b.timeline = timeline.data_ptr() if timeline is not None else None
    with torch.cuda.device(events.device):   # K0/K1 launch on the device that holds the batch
        _check(lib().gml_replay(C.byref(b)), "gml_replay")
    return stats


def gml_last_launch_count() -> int:
    return int(lib().gml_last_launch_count())


def gml_last_kernel_ms() -> float:
    return float(lib().gml_last_kernel_ms())


def gml_last_split_count() -> tuple[int, int]:
    """(units that completed as split units, split units re-run by the
    single-warp replay) of the last gml_replay on this thread"""
    r = C.c_uint32(0)
    n = lib().gml_last_split_count(C.byref(r))
    return int(n), int(r.value)


def stats_from_bytes(buf: np.ndarray) -> np.ndarray:
    """uint8 buffer of n * 272 bytes -> structured array of gml_stats_t."""
    return np.frombuffer(np.ascontiguousarray(buf).tobytes(), dtype=STATS_DTYPE)


def stats_dict(rec) -> dict:
    d = {}
    for name in STATS_DTYPE.names:
        if name.startswith("_"):
            continue
        v = rec[name]
        d[name] = [int(x) for x in v] if np.ndim(v) else int(v)
    return d


def _as_struct(d: dict) -> gml_stats_t:
    s = gml_stats_t()
    for k, v in d.items():
        if isinstance(v, list):
            getattr(s, k)[:] = v
        else:
            setattr(s, k, v)
    return s


def gml_utilization(stats: dict) -> float:
    return float(lib().gml_utilization(C.byref(_as_struct(stats))))


def gml_fragmentation(stats: dict) -> float:
    return float(lib().gml_fragmentation(C.byref(_as_struct(stats))))


# ------------------------------------------------------------ live allocator
class Allocator:
    """gml_create / gml_malloc / gml_free / gml_stats / gml_destroy."""

    def __init__(self, device: int, policy: dict):
        self._h = C.c_void_p(None)
        self._p = to_policy(policy)
        _check(lib().gml_create(int(device), C.byref(self._p), C.byref(self._h)), "gml_create")

    def malloc(self, nbytes: int) -> int:
        out = C.c_void_p(None)
        rc = lib().gml_malloc(self._h, int(nbytes), C.byref(out))
        _check(rc, "gml_malloc")
        return int(out.value)

    def free(self, ptr: int) -> None:
        _check(lib().gml_free(self._h, C.c_void_p(ptr)), "gml_free")

    def set_stream(self, stream) -> None:
        """Order StitchFree's deferred unmaps on `stream` (a torch.cuda.Stream or a raw handle)."""
        h = getattr(stream, "cuda_stream", stream)
        _check(lib().gml_set_stream(self._h, C.c_void_p(h)), "gml_set_stream")

    def trace(self, events: np.ndarray):
        """gml_live_trace: -> (status, n_done, records u64[n], ns u64[n])."""
        ev = np.ascontiguousarray(events, dtype=np.uint64)
        rec = np.zeros(max(len(ev), 1), np.uint64)
        ns = np.zeros(max(len(ev), 1), np.uint64)
        done = C.c_uint64(0)
        p = lambda a: a.ctypes.data_as(C.POINTER(C.c_uint64))
        rc = lib().gml_live_trace(self._h, p(ev), len(ev), p(rec), p(ns), C.byref(done))
        return rc, int(done.value), rec[:len(ev)], ns[:len(ev)]

    def stats(self) -> dict:
        s = gml_stats_t()
        _check(lib().gml_stats(self._h, C.byref(s)), "gml_stats")
        raw = np.frombuffer(bytes(s), dtype=STATS_DTYPE)[0]
        return stats_dict(raw)

    def driver_calls(self) -> list[int]:
        buf = (C.c_uint64 * 7)()
        _check(lib().gml_driver_calls(self._h, buf), "gml_driver_calls")
        return [int(x) for x in buf]

    def destroy(self) -> None:
        if self._h:
            _check(lib().gml_destroy(self._h), "gml_destroy")
            self._h = C.c_void_p(None)


def gml_cudamalloc_trace(device: int, events: np.ndarray):
    """-> (status, n_done, ns u64[n]) of the trace as cudaMalloc / cudaFree."""
    ev = np.ascontiguousarray(events, dtype=np.uint64)
    ns = np.zeros(max(len(ev), 1), np.uint64)
    done = C.c_uint64(0)
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_uint64))
    rc = lib().gml_cudamalloc_trace(int(device), p(ev), len(ev), p(ns), C.byref(done))
    return rc, int(done.value), ns[:len(ev)]


def gml_stream_copy(src: int, dst: int, nbytes: int, iters: int, stream=None) -> float:
    import torch
    ms = C.c_float(0)
    s = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
    _check(lib().gml_stream_copy(C.c_void_p(src), C.c_void_p(dst), int(nbytes), int(iters),
                                 C.c_void_p(s), C.byref(ms)), "gml_stream_copy")
    return float(ms.value)
