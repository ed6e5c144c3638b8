"""Synthetic workloads of SURVEY.md §8d for bench.py and the parity tests (host-side input generation,
the role the reference's rng.hpp input generator plays; not part of the device path).

* ``gaussian``: K, V, Q ~ N(0, 1), post-RoPE, rounded to nearest-even bf16.
* ``structured``: the same plus planted heavy hitters.  In every (sequence, layer) a set of
  n = k/4 prefix positions is chosen; at those positions the key of EVERY KV head g is shifted by
  delta_g = t * qbar_g / |qbar_g|^2, where qbar_g is the mean of the queries that score the column
  (the G q-heads of g over the collected verify rows).  The mean raw logit of those queries against a
  planted key then rises by exactly t, so the Collect-k score of a planted column rises by t (per-layer
  and per-KV-head modes alike).  t defaults to 3 sigma of a single logit, 3 * sqrt(d): top-k has a
  real tail to recover instead of Gaussian noise around a flat threshold.
"""
from __future__ import annotations

import math

import numpy as np

D = 128
DATA_KINDS = ("gaussian", "structured")


def heavy_hitter_positions(p: int, k: int, rng: np.random.Generator) -> np.ndarray:
    """n = k // 4 distinct positions in [0, p), ascending."""
    n = max(1, min(p, k // 4))
    return np.sort(rng.choice(p, size=n, replace=False)).astype(np.int64)


def plant_shift(q_rows: np.ndarray, t: float) -> np.ndarray:
    """delta with mean_r(q_r . delta) = t for the query rows q_rows [n][d]: t * qbar / |qbar|^2."""
    qbar = np.asarray(q_rows, np.float64).reshape(-1, q_rows.shape[-1]).mean(0)
    return (t * qbar / max(float(qbar @ qbar), 1e-30)).astype(np.float32)


def default_shift(d: int = D) -> float:
    return 3.0 * math.sqrt(d)


def plant_torch(K_chunk, pos0, planted_by_layer, deltas):
    """Add the planted shifts to one chunk of keys in place (torch, on the chunk's device).

    K_chunk: [n][L*Hkv][d] fp32 (tokens pos0 .. pos0+n-1 of one sequence), planted_by_layer: list of L
    ascending int64 numpy arrays, deltas: [L][Hkv][d] fp32 tensor on the same device."""
    import torch
    n = K_chunk.shape[0]
    L, Hkv, d = deltas.shape
    Kv = K_chunk.view(n, L, Hkv, d)
    for layer, pos in enumerate(planted_by_layer):
        lo, hi = np.searchsorted(pos, [pos0, pos0 + n])
        if hi > lo:
            rows = torch.as_tensor(pos[lo:hi] - pos0, device=K_chunk.device)
            Kv[rows, layer] += deltas[layer].unsqueeze(0)
    return K_chunk
