"""Batch x KV-head sharding across the GPUs of one node and the single exchange
step the path has.

The reference is single-process; sharding is new.  Units of work are independent
(sequence, KV head) pairs except for one thing: per-layer selection (the reference default,
selection.cpp:96 / SPEC.md:335) averages the raw logits of ALL q-heads of a layer, so when a
layer's KV heads live on different ranks their column sums must be combined before top-k.  The
verify kernel emits those sums as int64 fixed point (units of 2^-32), so the combination is an
integer all-reduce: exact and independent of the reduction order, hence a head-sharded selection is
bit-identical to the single-GPU one.  Per-KV-head selection needs no exchange at all.

Plumbing only: torch.distributed (NCCL on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

FX_SCALE = 2.0 ** 32  # units of the per-layer fixed-point column sums (kScoreFxScale in common.cuh)


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    seqs: tuple        # global sequence ids owned by this rank
    heads: range       # KV heads owned by this rank
    head_group: int    # ranks that share this rank's sequences (1 = pure batch sharding)

    @property
    def needs_score_exchange(self) -> bool:
        """Per-layer selection over KV heads split across ranks needs the one all-reduce."""
        return self.head_group > 1


def plan(batch: int, n_kv_heads: int, world: int, rank: int) -> Shard:
    """Shard `batch` sequences x `n_kv_heads` KV heads over `world` ranks.

    Batch first (no exchange): wb = gcd(batch, world) batch groups; the remaining factor wh =
    world / wb splits the KV heads (must divide n_kv_heads).  Ranks of one batch group are
    consecutive, so a head group is a contiguous rank range (one NCCL sub-communicator)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank/world out of range")
    wb = math.gcd(batch, world)
    wh = world // wb
    if n_kv_heads % wh:
        raise ValueError(f"cannot shard {batch} sequences x {n_kv_heads} KV heads over {world} ranks")
    bgrp, hgrp = divmod(rank, wh)
    per_b = batch // wb
    per_h = n_kv_heads // wh
    return Shard(rank, world, tuple(range(bgrp * per_b, (bgrp + 1) * per_b)),
                 range(hgrp * per_h, (hgrp + 1) * per_h), wh)


def plan_heads(batch: int, n_kv_heads: int, world: int, rank: int) -> Shard:
    """Shard the KV heads over ALL `world` ranks, every rank holding every sequence (the config-4
    style split: each GPU owns n_kv_heads / world heads of every sequence and their G q-heads).
    Per-layer selection then needs the exchange over the whole group."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank/world out of range")
    if n_kv_heads % world:
        raise ValueError(f"cannot split {n_kv_heads} KV heads over {world} ranks")
    per_h = n_kv_heads // world
    return Shard(rank, world, tuple(range(batch)), range(rank * per_h, (rank + 1) * per_h), world)


def head_group_ranks(shard: Shard) -> list:
    """Ranks that hold the other KV heads of this rank's sequences."""
    base = (shard.rank // shard.head_group) * shard.head_group
    return list(range(base, base + shard.head_group))


def exchange_layer_scores(fx, shard: Shard, group=None) -> None:
    """In-place sum of the per-layer int64 column sums over the head group (the §8e exchange).
    `fx` is the [B][ld] int64 tensor of one layer (Runner.layer_scores_tensor on the GPU)."""
    if not shard.needs_score_exchange:
        return
    import torch
    import torch.distributed as dist
    if fx.dtype != torch.int64:
        raise TypeError("per-layer score sums are int64 fixed point")
    dist.all_reduce(fx, op=dist.ReduceOp.SUM, group=group)


def to_fixed_point(col_sums_f32):
    """Host restatement of the kernel's conversion (verify_tc.cu): round-to-nearest of the fp32
    per-head column sum x 2^32, saturating to int64 (cvt.rni.s64.f32)."""
    import numpy as np
    x = np.asarray(col_sums_f32, np.float32).astype(np.float64) * FX_SCALE
    x = np.clip(np.rint(x), -2.0 ** 63, 2.0 ** 63 - 1024)
    return x.astype(np.int64)
