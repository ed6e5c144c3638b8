"""Shared helpers for the GPU parity tests: matched device/reference stores and error metrics."""
from __future__ import annotations

import numpy as np

from oracle.counter_rng import normal_bf16

D = 128


def rel_err_rows(gpu: np.ndarray, ref: np.ndarray) -> float:
    """max over rows of max|gpu-ref| / max|ref| (normwise per output vector)."""
    gpu = gpu.reshape(-1, gpu.shape[-1]).astype(np.float64)
    ref = ref.reshape(-1, ref.shape[-1]).astype(np.float64)
    den = np.maximum(np.abs(ref).max(-1), 1e-30)
    return float((np.abs(gpu - ref).max(-1) / den).max())


def rel_err_elem(gpu: np.ndarray, ref: np.ndarray, tau: float = 1e-3) -> float:
    """|gpu-ref| / max(|ref|, tau * max_row|ref|), max over elements."""
    gpu = gpu.reshape(-1, gpu.shape[-1]).astype(np.float64)
    ref = ref.reshape(-1, ref.shape[-1]).astype(np.float64)
    floor = tau * np.abs(ref).max(-1, keepdims=True)
    return float((np.abs(gpu - ref) / np.maximum(np.abs(ref), floor)).max())


def check_selection(gpu_idx, ref_scores, k, band_rel=2e-3, relative=False):
    """North-star index contract: |GPU| = k, GPU ⊇ {s > s_k + band}, GPU ⊆ {s >= s_k - band};
    band = band_rel * max(|s_k|, 1) (raw-logit scores) or band_rel * |s_k| (relative=True: softmax
    weights, whose scale is ~1/p)."""
    gpu = np.asarray(gpu_idx, np.int64)
    assert len(gpu) == k, (len(gpu), k)
    assert np.all(np.diff(gpu) > 0), "indices must be strictly increasing"
    if k == 0:
        return True
    s_k = np.sort(ref_scores)[::-1][k - 1]
    band = band_rel * (abs(s_k) if relative else max(abs(s_k), 1.0))
    must = np.nonzero(ref_scores > s_k + band)[0]
    allowed = np.nonzero(ref_scores >= s_k - band)[0]
    gs = set(gpu.tolist())
    assert set(must.tolist()) <= gs, "a clearly-selected column is missing"
    assert gs <= set(allowed.tolist()), "a clearly-rejected column was selected"
    return True


class Matched:
    """A device cache and a reference KvStore holding the same bf16-representable tokens."""

    def __init__(self, ref, L, Hkv, n_tokens, seed, max_context=None, page_size=256, n_seqs=1, lens=None):
        import torch

        from paper_2602_07223_b200 import Cache
        self.L, self.Hkv = L, Hkv
        max_context = max_context or (n_tokens + 64)
        self.cache = Cache(L, Hkv, D, max_context, max_seqs=n_seqs, page_size=page_size)
        self.refs = []
        lens = lens or [n_tokens] * n_seqs
        self.K, self.V = [], []
        for s in range(n_seqs):
            K = normal_bf16(seed + s, 1, (lens[s], L * Hkv, D))
            V = normal_bf16(seed + s, 2, (lens[s], L * Hkv, D))
            kv = ref.kv(L, Hkv, D, max_context)
            for t in range(lens[s]):
                kv.append(K[t], V[t])
            if lens[s]:
                self.cache.append(torch.from_numpy(K).cuda(), torch.from_numpy(V).cuda(), seq=s)
            self.refs.append(kv)
            self.K.append(K)
            self.V.append(V)
        torch.cuda.synchronize()


def to_dev_bf16(x: np.ndarray):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda().to(torch.bfloat16)
