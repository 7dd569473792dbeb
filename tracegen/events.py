"""Packed allocation-trace events.

This module is INPUT infrastructure shared by the oracle tests and the CUDA
path. It holds no allocator arithmetic: only the event encoding, a bookkeeping
validator and the slot assignment that turns logical tensor ids into reusable
handle slots.

Event word (u64, little-endian), one per malloc or free (SPEC.md L347-352,
"op: {malloc, free}; id; size"):

    bit 63        1 = free, 0 = malloc
    bits 40..62   slot (23 bits): the handle the event binds / unbinds
    bits 0..39    raw request bytes (malloc), 0 (free)
"""
from __future__ import annotations

import heapq
import json
from typing import Iterable, Sequence

import numpy as np

FREE_BIT = np.uint64(1) << np.uint64(63)
SLOT_SHIFT = 40
SLOT_BITS = 23
SIZE_BITS = 40
MAX_SLOT = (1 << SLOT_BITS) - 1
MAX_SIZE = (1 << SIZE_BITS) - 1


def enc_malloc(slot: int, size: int) -> int:
    if not (0 <= slot <= MAX_SLOT):
        raise ValueError(f"slot {slot} out of range")
    if not (0 < size <= MAX_SIZE):
        raise ValueError(f"size {size} out of range")
    return (slot << SLOT_SHIFT) | size


def enc_free(slot: int) -> int:
    if not (0 <= slot <= MAX_SLOT):
        raise ValueError(f"slot {slot} out of range")
    return (1 << 63) | (slot << SLOT_SHIFT)


def decode(ev: int) -> tuple[bool, int, int]:
    """-> (is_free, slot, size)."""
    ev = int(ev)
    return bool(ev >> 63), (ev >> SLOT_SHIFT) & MAX_SLOT, ev & MAX_SIZE


def pack(ops: Iterable[tuple[str, int, int]]) -> np.ndarray:
    """[('m', slot, size) | ('f', slot, 0)] -> uint64 array."""
    out = []
    for op, slot, size in ops:
        out.append(enc_malloc(slot, size) if op == "m" else enc_free(slot))
    return np.array(out, dtype=np.uint64)


def unpack(events: np.ndarray) -> list[tuple[str, int, int]]:
    res = []
    for ev in events.tolist():
        f, slot, size = decode(ev)
        res.append(("f" if f else "m", slot, size))
    return res


class TraceError(ValueError):
    pass


def validate(events: np.ndarray) -> int:
    """Bookkeeping check (SURVEY §8(b) 'Trace validation'): every free names a
    live slot, every malloc slot is free, sizes > 0, free words carry size 0.
    Returns max_slots (= 1 + the largest slot used, 0 for an empty trace)."""
    live = set()
    max_slot = -1
    ev = np.asarray(events, dtype=np.uint64)
    is_free = (ev >> np.uint64(63)).astype(bool)
    slots = ((ev >> np.uint64(SLOT_SHIFT)) & np.uint64(MAX_SLOT)).astype(np.int64)
    sizes = (ev & np.uint64(MAX_SIZE)).astype(np.int64)
    for i in range(len(ev)):
        s = int(slots[i])
        if is_free[i]:
            if sizes[i] != 0:
                raise TraceError(f"event {i}: free carries a size")
            if s not in live:
                raise TraceError(f"event {i}: free of slot {s} which is not live")
            live.remove(s)
        else:
            if sizes[i] == 0:
                raise TraceError(f"event {i}: zero-byte malloc")
            if s in live:
                raise TraceError(f"event {i}: malloc into live slot {s}")
            live.add(s)
        if s > max_slot:
            max_slot = s
    return max_slot + 1


class SlotAssigner:
    """Maps logical tensor ids to the lowest free slot (so max_slots equals the
    peak number of live tensors)."""

    def __init__(self):
        self._free: list[int] = []
        self._next = 0
        self._of: dict = {}
        self.events: list[int] = []

    def malloc(self, tid, size: int) -> None:
        if tid in self._of:
            raise TraceError(f"tensor {tid!r} already live")
        if self._free:
            s = heapq.heappop(self._free)
        else:
            s = self._next
            self._next += 1
        self._of[tid] = s
        self.events.append(enc_malloc(s, int(size)))

    def free(self, tid) -> None:
        s = self._of.pop(tid)
        heapq.heappush(self._free, s)
        self.events.append(enc_free(s))

    def live(self) -> list:
        return list(self._of.keys())

    def is_live(self, tid) -> bool:
        return tid in self._of

    def array(self) -> np.ndarray:
        return np.array(self.events, dtype=np.uint64)


def to_jsonl(events: np.ndarray) -> str:
    """SPEC.md L407 interop: {"seq", "op", "id", "size"} per line. The id is
    the slot plus a generation counter so that ids are never reused."""
    gen: dict[int, int] = {}
    lines = []
    for seq, (op, slot, size) in enumerate(unpack(events)):
        if op == "m":
            g = gen.get(slot, -1) + 1
            gen[slot] = g
            tid = (g << SLOT_BITS) | slot
            lines.append(json.dumps({"seq": seq, "op": "malloc", "id": tid, "size": size}))
        else:
            tid = (gen[slot] << SLOT_BITS) | slot
            lines.append(json.dumps({"seq": seq, "op": "free", "id": tid}))
    return "\n".join(lines) + ("\n" if lines else "")


def from_jsonl(text: str) -> np.ndarray:
    sa = SlotAssigner()
    last = -1
    for ln, line in enumerate(text.splitlines(), 1):
        if not line.strip():
            continue
        obj = json.loads(line)
        keys = set(obj)
        if obj.get("op") == "malloc":
            if keys != {"seq", "op", "id", "size"}:
                raise TraceError(f"line {ln}: bad fields {sorted(keys)}")
        elif obj.get("op") == "free":
            if keys != {"seq", "op", "id"}:
                raise TraceError(f"line {ln}: bad fields {sorted(keys)}")
        else:
            raise TraceError(f"line {ln}: bad op")
        if obj["seq"] <= last:
            raise TraceError(f"line {ln}: seq not increasing")
        last = obj["seq"]
        try:
            if obj["op"] == "malloc":
                sa.malloc(obj["id"], obj["size"])
            else:
                sa.free(obj["id"])
        except KeyError:
            raise TraceError(f"line {ln}: free of unknown id") from None
    return sa.array()


def concat(traces: Sequence[np.ndarray]) -> tuple[np.ndarray, np.ndarray]:
    """Batch layout for gml_replay: all traces back to back + n+1 offsets."""
    offs = np.zeros(len(traces) + 1, dtype=np.uint64)
    for i, t in enumerate(traces):
        offs[i + 1] = offs[i] + np.uint64(len(t))
    ev = np.concatenate([np.asarray(t, dtype=np.uint64) for t in traces]) if traces else np.zeros(0, np.uint64)
    return ev, offs
