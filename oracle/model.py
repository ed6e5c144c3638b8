"""Model-side producer restatement (RMSNorm -> Q/K/V projection -> RoPE) — TEST INFRASTRUCTURE ONLY,
the checker for csrc/qkv.cu.

PARITY UNPINNED against code: the reference ships the weights layout (weights.hpp:20-30) and config
(config.hpp:22-35) but not the forward; this restates SPEC forward, "RMS
normalization" and apply_rope in float64 and is pinned on the SPEC's
apply_rope examples (tests/test_oracle.py).  RoPE pair conventions: style 0 = half-split pairs
(i, i + d/2), style 1 = interleaved pairs (2j, 2j+1); pair j rotates by pos * theta^(-2j/d).

Only tests/, __graft_entry__.smoke() and bench.py may import this module.
"""
from __future__ import annotations

import numpy as np


def rms_norm(x, gain, eps):
    """x / sqrt(mean(x^2) + eps) * gain, float64 (per row)."""
    x = np.asarray(x, dtype=np.float64)
    r = 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)
    return x * r * np.asarray(gain, dtype=np.float64)


def apply_rope(v, position, theta=10000.0, style=0):
    """Rotate one head vector (last axis = head_dim, even) by `position`."""
    v = np.asarray(v, dtype=np.float64)
    d = v.shape[-1]
    if d % 2:
        raise ValueError("apply_rope: head_dim must be even")
    j = np.arange(d // 2, dtype=np.float64)
    ang = np.float64(position) * theta ** (-2.0 * j / d)
    c, s = np.cos(ang), np.sin(ang)
    out = np.empty_like(v)
    if style == 0:
        a, b = v[..., :d // 2], v[..., d // 2:]
        out[..., :d // 2] = a * c - b * s
        out[..., d // 2:] = b * c + a * s
    else:
        a, b = v[..., 0::2], v[..., 1::2]
        out[..., 0::2] = a * c - b * s
        out[..., 1::2] = b * c + a * s
    return out


def qkv_project(x, w_qkv, gain, Hq, Hkv, positions, eps=1e-5, theta=10000.0, style=0):
    """x [B][rows][D]; w_qkv [(Hq+2Hkv)*128][D] (rows of wq^T, wk^T, wv^T); positions [B] (row 0).
    Returns float64 q [B][Hq][rows][128], k [B][rows][Hkv][128], v [B][rows][Hkv][128]."""
    x = np.asarray(x, dtype=np.float64)
    B, rows, D = x.shape
    h = rms_norm(x, gain, eps)
    y = h @ np.asarray(w_qkv, dtype=np.float64).T  # [B][rows][(Hq+2Hkv)*128]
    y = y.reshape(B, rows, Hq + 2 * Hkv, 128)
    for b in range(B):
        for r in range(rows):
            pos = int(positions[b]) + r
            y[b, r, :Hq + Hkv] = apply_rope(y[b, r, :Hq + Hkv], pos, theta, style)
    q = y[:, :, :Hq].transpose(0, 2, 1, 3)
    return q, y[:, :, Hq:Hq + Hkv], y[:, :, Hq + Hkv:]
