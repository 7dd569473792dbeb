"""Seeded synthetic allocation traces (input infrastructure shared by the
oracle tests and the CUDA path; holds none of the allocator's arithmetic)."""
from .events import (enc_malloc, enc_free, decode, pack, unpack, validate, concat,
                     to_jsonl, from_jsonl, SlotAssigner, TraceError)
from . import synth
from . import snapshot
