"""Policy-variant table V0-V7: configuration only.

A policy is a plain dict with the fields of gml_policy (include/gml.h). Both
the oracle binding (tests/oracle_lib.py) and the product binding
(paper_2401_08156_b200/gml.py) marshal these dicts into their own structs.
"""
from __future__ import annotations

MiB = 1 << 20
GiB = 1 << 30

BFC_TORCH, BFC_EXACT, GMLAKE = 0, 1, 2
F_S1_PBLOCK_FIRST, F_NO_COMPANION, F_SPLIT_INVALIDATES, F_REMAINDER_RULE = 1, 2, 4, 8


def policy(kind: int = GMLAKE, flags: int = 0, capacity: int = 80 * GiB, chunk: int = 2 * MiB,
           small_threshold: int = 2 * MiB, frag_limit: int = 128 * MiB,
           spool_max_entries: int = 4096, spool_max_inactive_bytes: int | None = None) -> dict:
    """Defaults: capacity 80 GiB (A100-80GB testbed), 2 MiB
    chunk, 2 MiB small-path threshold,
    128 MiB fragmentation limit, sPool caps (D17)."""
    return dict(kind=kind, flags=flags, capacity_bytes=capacity, chunk_bytes=chunk,
                small_threshold_bytes=small_threshold, frag_limit_bytes=frag_limit,
                spool_max_entries=spool_max_entries,
                spool_max_inactive_bytes=capacity if spool_max_inactive_bytes is None
                else spool_max_inactive_bytes)


def variants(capacity: int = 80 * GiB) -> list[dict]:
    """V0..V7 in order."""
    return [
        policy(BFC_TORCH, capacity=capacity),                               # V0 PyTorch caching allocator
        policy(BFC_EXACT, capacity=capacity),                               # V1 BFC-exact
        policy(GMLAKE, capacity=capacity),                                  # V2 GMLake default
        policy(GMLAKE, capacity=capacity, frag_limit=2 * MiB),              # V3 limit = chunk
        policy(GMLAKE, F_REMAINDER_RULE, capacity=capacity),                # V4
        policy(GMLAKE, F_SPLIT_INVALIDATES, capacity=capacity),             # V5
        policy(GMLAKE, F_NO_COMPANION, capacity=capacity),                  # V6
        policy(GMLAKE, capacity=capacity, spool_max_entries=64),            # V7 small sPool
    ]


VARIANT_NAMES = ["V0 bfc-torch", "V1 bfc-exact", "V2 gmlake", "V3 gmlake-limit2M",
                 "V4 remainder-rule", "V5 split-invalidates", "V6 no-companion", "V7 spool64"]
