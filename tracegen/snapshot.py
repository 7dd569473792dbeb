"""Real-trace ingestion: a PyTorch CUDA memory snapshot
(`torch.cuda.memory._record_memory_history()` + `torch.cuda.memory._snapshot()`)
-> packed allocation events (events.py). Input infrastructure only: no
allocator arithmetic.

The snapshot's `device_traces[d]` lists trace entries in program order; an
entry is a dict with `action` in {alloc, free_requested, free_completed,
segment_alloc, segment_free, segment_map, segment_unmap, snapshot, oom},
`addr`, `size` and `stream`. Each `alloc` becomes a malloc of `size` bytes on
a new tensor id (the address, live until freed); the matching free becomes a
free. Frees of addresses allocated before recording started are dropped;
tensors still live at the end stay live (no implicit frees, D28). Segment
events are the caching allocator's own cudaMalloc/cudaFree calls -- the very
decisions GMLake replaces -- and are not part of the request stream.

`free_at="free_requested"` (default) frees when the program releases the
tensor; "free_completed" when the caching allocator could reuse it (later
when the block was used on another stream).
"""
from __future__ import annotations

import numpy as np

from .events import SlotAssigner

_FREE_ACTIONS = ("free_requested", "free_completed")


def from_snapshot(snap: dict, device: int = 0, free_at: str = "free_requested") -> np.ndarray:
    if free_at not in _FREE_ACTIONS:
        raise ValueError(f"free_at must be one of {_FREE_ACTIONS}")
    traces = snap.get("device_traces", [])
    entries = traces[device] if device < len(traces) else []
    sa = SlotAssigner()
    live: dict[int, int] = {}
    serial = 0
    for e in entries:
        act = e.get("action")
        if act == "alloc":
            addr = int(e["addr"])
            size = int(e["size"])
            if size <= 0:
                continue
            if addr in live:                 # address reused without a recorded free
                sa.free(live.pop(addr))
            live[addr] = serial
            sa.malloc(serial, size)
            serial += 1
        elif act == free_at:
            tid = live.pop(int(e["addr"]), None)
            if tid is not None:
                sa.free(tid)
    return np.array(sa.events, dtype=np.uint64)


def load(path: str, device: int = 0, free_at: str = "free_requested") -> np.ndarray:
    """Events of a pickled snapshot file (torch.cuda.memory._dump_snapshot)."""
    import pickle
    with open(path, "rb") as fh:
        return from_snapshot(pickle.load(fh), device, free_at)
