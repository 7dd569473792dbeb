"""B200-native GMLake allocation engine (arXiv 2401.08156).

The product is libgml.so (C ABI, include/gml.h): batched trace replay on
sm_100a (gml_replay) and a live VMM allocator (gml_malloc / gml_free /
gml_stats). This package is its thin Python binding.
"""
from . import gml  # noqa: F401  (fails loudly at call time if libgml.so is missing)

__all__ = ["gml"]
