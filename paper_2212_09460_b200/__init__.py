"""B200-native (sm_100a) lane-detection hot path of arXiv 2212.09460.

Public API: the Python binding in :mod:`paper_2212_09460_b200.ld`, with the
same names as the C ABI in ``include/ld.h``.  The CUDA library is loaded on
first use and its absence is an error (there is no CPU fallback).
"""
from . import synth  # noqa: F401  (seeded inputs only; no method arithmetic)
