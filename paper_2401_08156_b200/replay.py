"""Batch helpers around gml_replay: pack traces into device buffers, run the
replay, decode the outputs. Marshalling only -- the replay runs in K1."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import gml


@dataclass
class DeviceBatch:
    events: "torch.Tensor"         # int64 [total] (packed u64 events)
    offsets: "torch.Tensor"        # int64 [T + 1]
    n_traces: int
    total: int

    @property
    def bytes(self) -> int:
        return 8 * self.total + 8 * (self.n_traces + 1)


def upload(traces, device="cuda", pin: bool = True) -> DeviceBatch:
    import torch
    offs = np.zeros(len(traces) + 1, dtype=np.int64)
    for i, t in enumerate(traces):
        offs[i + 1] = offs[i] + len(t)
    ev = np.concatenate([np.asarray(t, dtype=np.uint64) for t in traces]).view(np.int64)
    te = torch.from_numpy(ev)
    to = torch.from_numpy(offs)
    if pin:
        te, to = te.pin_memory(), to.pin_memory()
    return DeviceBatch(te.to(device, non_blocking=True), to.to(device, non_blocking=True),
                       len(traces), int(offs[-1]))


def run(batch: DeviceBatch, policies, with_assignments: bool = True, stream=None, caps=None,
        assignments=None, stats=None, timeline=None):
    """-> (assignments int64 tensor [P, total] or None, stats uint8 tensor);
    `timeline` (optional int64 tensor [P, total, 2]) receives (active,
    reserved) after each event."""
    import torch
    dev = batch.events.device
    if with_assignments and assignments is None:
        assignments = torch.empty((len(policies), max(batch.total, 1)), dtype=torch.int64, device=dev)
    st = gml.gml_replay(batch.events, batch.offsets, policies,
                        assignments if with_assignments else None, stats, stream, caps, timeline)
    return assignments, st


def decode_stats(stats_tensor, n_traces: int, n_policies: int) -> list[list[dict]]:
    arr = gml.stats_from_bytes(stats_tensor.cpu().numpy())
    return [[gml.stats_dict(arr[t * n_policies + p]) for p in range(n_policies)] for t in range(n_traces)]


def tight_caps(stats: list[list[dict]], slack: float = 1.0) -> np.ndarray:
    """Table hints for a re-run from the maxima a previous replay observed
    (the same batch replays identically; intervals are estimated as 4 per
    sBlock -- an underestimate only costs an overflow re-run)."""
    rows = []
    for per_t in stats:
        for s in per_t:
            p = max(64, int(s["max_pblocks"] * slack) + 8)
            sb = max(64, int(s["max_sblocks"] * slack) + 8)
            rows.append((p, sb, max(128, 4 * sb), max(64, int(s["max_bfc_blocks"] * slack) + 8)))
    return np.ascontiguousarray(np.array(rows, dtype=np.uint32))
