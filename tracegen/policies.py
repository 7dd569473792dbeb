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
F_LIMIT_GATES_REQUEST = 16    # D8': requests below the fragmentation limit take the small path


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
    """V0..V7 in order. V2 is the GMLake default under reading D8' (requests
    below the 128 MiB fragmentation limit take the small path, PAPER.md
    L571 + L322); V4-V7 are the literal-D8 family (the limit only filters
    candidate blocks), which drives the VMM mechanisms (Split, Stitch,
    StitchFree) the gate routes away from: V7 is literal D8 alone (round 1's
    default), V4-V6 add one ambiguity switch each."""
    gate = F_LIMIT_GATES_REQUEST
    return [
        policy(BFC_TORCH, capacity=capacity),                               # V0 PyTorch caching allocator
        policy(BFC_EXACT, capacity=capacity),                               # V1 BFC-exact
        policy(GMLAKE, gate, capacity=capacity),                            # V2 GMLake default (D8')
        policy(GMLAKE, gate, capacity=capacity, frag_limit=2 * MiB),        # V3 limit = chunk
        policy(GMLAKE, F_REMAINDER_RULE, capacity=capacity),                # V4 literal + REMAINDER_RULE
        policy(GMLAKE, F_SPLIT_INVALIDATES, capacity=capacity),             # V5 literal + SPLIT_INVALIDATES
        policy(GMLAKE, F_NO_COMPANION, capacity=capacity),                  # V6 literal + NO_COMPANION
        policy(GMLAKE, capacity=capacity),                                  # V7 literal D8
    ]


def spool64(capacity: int = 80 * GiB) -> dict:
    """Literal D8 with a 64-entry sPool (count-cap StitchFree at scale; the
    round-1 V7, kept as a parity case)."""
    return policy(GMLAKE, capacity=capacity, spool_max_entries=64)


VARIANT_NAMES = ["V0 bfc-torch", "V1 bfc-exact", "V2 gmlake", "V3 gmlake-limit2M",
                 "V4 literal+remainder-rule", "V5 literal+split-invalidates", "V6 literal+no-companion",
                 "V7 gmlake-literal-D8"]
