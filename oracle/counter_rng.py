"""Vectorised numpy port of the reference CounterRng (rng.hpp:17-62) — TEST INFRASTRUCTURE ONLY.

Used to generate the synthetic Q/K/V inputs of the parity tests (SURVEY.md §8d "Synthetic
inputs"): streams are split with derive(label), draws are addressable by counter, normals use
Box-Muller on two 53-bit uniforms, then values are rounded to bf16 so the device (bf16) and the
oracle (fp32) see identical numbers.
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
SEED_TAG = 0x537065634174746E
CHILD_TAG = 0xA5A5A5A5DEADBEEF


def mix64(z):
    """rng.hpp:53-58 on python ints or uint64 arrays."""
    if isinstance(z, np.ndarray):
        with np.errstate(over="ignore"):
            z = z + np.uint64(GOLDEN)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            return z ^ (z >> np.uint64(31))
    z = (z + GOLDEN) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


class CounterRng:
    def __init__(self, key: int):
        self.key = key & M64

    @staticmethod
    def seeded(seed: int) -> "CounterRng":
        return CounterRng(mix64((seed ^ SEED_TAG) & M64))

    def derive(self, label: int) -> "CounterRng":
        return CounterRng(mix64(self.key ^ mix64((label + CHILD_TAG) & M64)))

    def at(self, i):
        if isinstance(i, np.ndarray):
            with np.errstate(over="ignore"):
                return mix64(np.uint64(self.key) + (i.astype(np.uint64) + np.uint64(1)) * np.uint64(GOLDEN))
        return mix64((self.key + (i + 1) * GOLDEN) & M64)

    def normals(self, n: int) -> np.ndarray:
        """First n normal() draws of a fresh stream (rng.hpp:40-45)."""
        c = np.arange(2 * n, dtype=np.uint64)
        u = (self.at(c) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        u1, u2 = u[0::2], u[1::2]
        u1 = np.where(u1 <= 0.0, 2.0 ** -53, u1)
        return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def bf16_round(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    r = (((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16).astype(np.uint32)
    return np.where(np.isnan(x), x, r.view(np.float32))


def normal_bf16(seed: int, label: int, shape, scale: float = 1.0) -> np.ndarray:
    """bf16-representable fp32 normals from stream seeded(seed).derive(label)."""
    n = int(np.prod(shape))
    v = CounterRng.seeded(seed).derive(label).normals(n) * scale
    return bf16_round(v.astype(np.float32)).reshape(shape)
