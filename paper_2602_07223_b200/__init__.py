"""B200-native SpecAttn hot path (verify-attention -> top-k KV selection -> sparse draft attention,
plus the paged KV cache), exposed through the C ABI in include/specattn_b200.h.

The product is lib/libspecattn_b200.so (hand-written sm_100a CUDA + C++ host).  This package is a
thin ctypes binding used by tests/ and bench.py; it never falls back to a CPU path — if the
shared library is missing or no CUDA device is present, every entry point raises.
"""
from ._lib import (  # noqa: F401
    ALL_DRAFT, COLLECT2, COLLECT2_WEIGHTS, LAST_ACCEPTED, QUEST_LIKE, WINDOW, PER_KV_HEAD, PER_LAYER, PHASE_DRAFT, PHASE_SELECT,
    PHASE_VERIFY, Cache, Comm, QkvProjection, Runner, SpecAttnError, accept, build, lib, lib_path, selection_k,
)

__all__ = ["accept", "QkvProjection", "Cache", "Comm", "Runner", "SpecAttnError", "build", "lib", "lib_path", "selection_k", "COLLECT2", "ALL_DRAFT",
           "LAST_ACCEPTED", "COLLECT2_WEIGHTS", "QUEST_LIKE", "WINDOW", "PER_LAYER", "PER_KV_HEAD", "PHASE_VERIFY", "PHASE_SELECT", "PHASE_DRAFT"]
