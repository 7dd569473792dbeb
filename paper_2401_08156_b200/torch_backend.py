"""GMLake as PyTorch's CUDA allocator: the paper's
deployment mode -- "integrate it into the caching allocator of PyTorch"
(PAPER.md L578), transparent to the training program (L470-473).

    from paper_2401_08156_b200 import torch_backend
    torch_backend.enable()            # before the first CUDA allocation
    ... train as usual ...
    torch_backend.stats()             # gml_stats of the device's allocator

Every tensor allocation then goes through libgml.so's gml_torch_malloc /
gml_torch_free (csrc/torch_alloc.cu) -> the live allocator (csrc/live.cu):
the same engine (policy.cuh) as the GPU replay, issuing cuMemCreate /
cuMemMap / cuMemSetAccess for Alloc and Stitch. Marshalling only.
"""
from __future__ import annotations

from . import gml

_enabled = False


def enable(policy: dict | None = None) -> None:
    """Route this process's CUDA tensor allocations through GMLake. Must run
    before any CUDA memory is allocated (PyTorch allows one switch)."""
    global _enabled
    import torch
    if _enabled:
        return
    if policy is not None:
        gml._check(gml.lib().gml_torch_configure(gml.to_policy(policy)), "gml_torch_configure")
    alloc = torch.cuda.memory.CUDAPluggableAllocator(str(gml.LIB_PATH), "gml_torch_malloc", "gml_torch_free")
    torch.cuda.memory.change_current_allocator(alloc)
    _enabled = True


def stats(device: int = 0) -> dict:
    """gml_stats of the allocator serving `device` (a dict, see gml.h)."""
    import ctypes as C

    import numpy as np
    st = gml.gml_stats_t()
    gml._check(gml.lib().gml_torch_stats(device, C.byref(st)), "gml_torch_stats")
    return gml.stats_dict(gml.stats_from_bytes(np.frombuffer(bytes(st), dtype=np.uint8))[0])
