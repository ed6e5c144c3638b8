"""Verification acceptance (modified rejection sampling) — TEST INFRASTRUCTURE ONLY, the checker
for csrc/accept.cu.

PARITY UNPINNED against code: the reference ships no speculation code; this
restates the SPEC contract speculation::verify and residual_distribution
 and is pinned on the SPEC's own known-answer examples (tests/test_oracle.py).

The sampling arithmetic mirrors accept.cu exactly so GPU parity is bit-exact: ratios and
max(0, p - q) in fp32, prefix sums in float64 in block_sample's fixed order (32 contiguous ranges,
each summed by a warp in rounds of 32 - lane sums over rounds, butterfly to the range total - and
totalled in order; the picked range split again into 32 sub-ranges the same way; the picked
sub-range rescanned with an inclusive warp scan), target = u * total, smallest token whose
inclusive prefix exceeds the target.

Only tests/, __graft_entry__.smoke() and bench.py may import this module.
"""
from __future__ import annotations

import numpy as np

WARPS = 32  # accept.cu: 1024 threads = 32 warps, each owning a contiguous range of the vocabulary


def residual_distribution(p, q):
    """normalize(max(0, p - q)); p == q exactly is rejected (ValueError)."""
    p = np.asarray(p, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    r = np.maximum(0.0, p - q)
    s = r.sum()
    if s <= 0.0:
        raise ValueError("residual_distribution: p == q, rejection impossible")
    return r / s


def _butterfly_sum(x):
    """Sum of 32 lane values in the order of a __shfl_xor butterfly (offsets 16, 8, 4, 2, 1)."""
    v = list(x)
    for off in (16, 8, 4, 2, 1):
        v = [v[l] + v[l ^ off] for l in range(32)]
    return v[0]


def _warp_scan(x):
    """Inclusive Hillis-Steele scan of 32 lane values (shfl_up offsets 1, 2, 4, 8, 16)."""
    v = list(x)
    for off in (1, 2, 4, 8, 16):
        v = [v[l] + v[l - off] if l >= off else v[l] for l in range(32)]
    return v


def _range_sum(w, lo, hi):
    lanes = [0.0] * 32
    for i in range(lo, hi):
        lanes[(i - lo) % 32] += float(w[i])
    return _butterfly_sum(lanes)


def _pick(part, run, target):
    run0 = run
    for t, x in enumerate(part):
        if run + x > target:
            return t, run
        run += x
    c = 0
    for t, x in enumerate(part):
        if x > 0.0:
            c = t
    run = run0
    for x in part[:c]:
        run += x
    return c, run


def _ceil32(n):
    return (n + 31) // 32 * 32


def inverse_cdf(w, u):
    """accept.cu block_sample: w float64 weights >= 0, u in [0,1)."""
    w = np.asarray(w, dtype=np.float64)
    V = w.shape[0]
    per1 = _ceil32(-(-V // WARPS))
    part = [_range_sum(w, min(V, k * per1), min(V, k * per1 + per1)) for k in range(WARPS)]
    total = 0.0
    for x in part:
        total += x
    target = u * total
    c1, base = _pick(part, 0.0, target)
    lo1, hi1 = c1 * per1, min(V, c1 * per1 + per1)
    per2 = _ceil32(-(-per1 // WARPS))
    part2 = []
    for k in range(WARPS):
        lo = min(hi1, lo1 + k * per2)
        part2.append(_range_sum(w, lo, min(hi1, lo + per2)))
    c2, base = _pick(part2, base, target)
    lo = min(hi1, lo1 + c2 * per2)
    hi = min(hi1, lo + per2)
    last_mass = -1
    for i0 in range(lo, hi, 32):
        e = [float(w[i]) if i < hi else 0.0 for i in range(i0, i0 + 32)]
        v = _warp_scan(e)
        for l in range(32):
            if e[l] > 0.0:
                last_mass = i0 + l
        for l in range(32):
            if base + v[l] > target:
                return i0 + l
        base += v[31]
    return last_mass


def argmax_lower(row):
    """argmax with ties to the lower token id."""
    return int(np.argmax(np.asarray(row)))  # numpy returns the first maximal index


def accept(p, draft, q=None, u=None, greedy=False):
    """One sequence: p [g+1][V] f32, q [g][V] f32, draft [g], u [g+1] f32.
    Returns (accepted a, emitted list of a+1 tokens)."""
    p = np.asarray(p, dtype=np.float32)
    g = p.shape[0] - 1
    out = []
    for t in range(g):
        x = int(draft[t])
        if greedy:
            am = argmax_lower(p[t])
            if x != am:
                return t, out + [am]
        else:
            qt = np.asarray(q[t], dtype=np.float32)
            ratio = np.float32(p[t][x]) / np.float32(qt[x])
            if not np.float32(u[t]) < min(np.float32(1.0), ratio):
                w = np.maximum(np.float32(0.0), p[t] - qt).astype(np.float64)
                return t, out + [inverse_cdf(w, float(np.float32(u[g])))]
        out.append(x)
    bonus = argmax_lower(p[g]) if greedy else inverse_cdf(p[g].astype(np.float64), float(np.float32(u[g])))
    return g, out + [bonus]
