"""Verification acceptance (modified rejection sampling) — TEST INFRASTRUCTURE ONLY, the checker
for csrc/accept.cu.

PARITY UNPINNED against code: the reference ships no speculation code; this
restates the SPEC contract speculation::verify and residual_distribution
 and is pinned on the SPEC's own known-answer examples (tests/test_oracle.py).

The sampling arithmetic mirrors accept.cu exactly so GPU parity is bit-exact: ratios and
max(0, p - q) in fp32, prefix sums in float64 over ceil(V/1024)-token chunks (sequential inside a
chunk, then over chunk totals in order), target = u * total, smallest token whose inclusive
prefix exceeds the target.

Only tests/, __graft_entry__.smoke() and bench.py may import this module.
"""
from __future__ import annotations

import numpy as np

THREADS = 1024  # accept.cu kAccThreads: the chunking of the prefix sums


def residual_distribution(p, q):
    """normalize(max(0, p - q)); p == q exactly is rejected (ValueError)."""
    p = np.asarray(p, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    r = np.maximum(0.0, p - q)
    s = r.sum()
    if s <= 0.0:
        raise ValueError("residual_distribution: p == q, rejection impossible")
    return r / s


def inverse_cdf(w, u):
    """accept.cu block_sample: w float64 weights >= 0, u in [0,1)."""
    w = np.asarray(w, dtype=np.float64)
    V = w.shape[0]
    per = -(-V // THREADS)
    chunks = [w[t * per:min(V, (t + 1) * per)] for t in range(THREADS) if t * per < V]
    part = [float(np.cumsum(c)[-1]) if len(c) else 0.0 for c in chunks]
    part += [0.0] * (THREADS - len(part))
    total = 0.0
    for x in part:
        total += x
    target = u * total
    run, c = 0.0, -1
    for t, x in enumerate(part):
        if run + x > target:
            c = t
            break
        run += x
    if c < 0:
        c = max(t for t, x in enumerate(part) if x > 0.0)
        run = 0.0
        for x in part[:c]:
            run += x
    r = -1
    for i in range(c * per, min(V, (c + 1) * per)):
        run += w[i]
        if w[i] > 0.0:
            r = i
        if run > target:
            return i
    return r


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
