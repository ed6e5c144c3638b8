"""Multi-process (gloo, world_size 2, CPU) tests of the sharding plan and the per-layer score
exchange: KV heads split over two ranks, each rank's fixed-point column sums of its
own heads all-reduced, then top-k — must equal the single-process selection over all heads."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2602_07223_b200.shard import head_group_ranks, plan


def test_plan_prefers_batch_then_heads():
    s = [plan(16, 8, 8, r) for r in range(8)]
    assert all(x.head_group == 1 and len(x.seqs) == 2 and x.heads == range(8) for x in s)
    s = [plan(4, 8, 8, r) for r in range(8)]  # config 4 shape: batch 4 x heads 2
    assert all(x.head_group == 2 and len(x.seqs) == 1 and len(x.heads) == 4 for x in s)
    assert sorted((x.seqs, x.heads.start) for x in s) == sorted({(x.seqs, x.heads.start) for x in s})
    s = [plan(1, 8, 8, r) for r in range(8)]  # batch 1: pure KV-head sharding
    assert [x.heads.start for x in s] == list(range(8)) and head_group_ranks(s[3]) == list(range(8))
    with pytest.raises(ValueError):
        plan(1, 8, 3, 0)


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, logits, G, rows, out_q):
    import torch
    import torch.distributed as dist

    from paper_2602_07223_b200.shard import exchange_layer_scores, plan, to_fixed_point
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        Hq, R, p = logits.shape
        sh = plan(1, Hq // G, world, rank)
        # this rank's fp32 per-KV-head column sums of rows {1, R} (what its verify kernel writes) ...
        local = np.zeros(p, np.int64)
        for g in sh.heads:
            s = logits[g * G:(g + 1) * G][:, rows, :].astype(np.float32).sum((0, 1), dtype=np.float32)
            local += to_fixed_point(s)
        fx = torch.from_numpy(local.reshape(1, p).copy())
        exchange_layer_scores(fx, sh)  # ... summed over the head group: exact int64 all-reduce
        out_q.put((rank, fx.numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_head_sharded_selection_equals_single_process(oracle):
    from paper_2602_07223_b200.shard import to_fixed_point
    from oracle.counter_rng import normal_bf16
    from oracle.pyoracle import COLLECT2
    Hkv, G, R, p, world = 4, 4, 5, 700, 2
    Hq = Hkv * G
    logits = normal_bf16(91, 1, (Hq, R, p), scale=8.0)
    rows = [0, R - 1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, logits, G, rows, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    # every rank holds the same, complete sums
    assert np.array_equal(res[0], res[1])
    single = np.zeros(p, np.int64)
    for g in range(Hkv):
        single += to_fixed_point(logits[g * G:(g + 1) * G][:, rows, :].astype(np.float32).sum((0, 1), dtype=np.float32))
    assert np.array_equal(res[0][0], single)  # bit-identical to one process holding all heads
    # top-k of the exchanged sums == the reference's select_collect2 over all heads
    k = oracle.selection_k(0.07, p, 16)
    got = oracle.topk_indices(res[0][0].astype(np.float64), k)
    want = oracle.select(COLLECT2, logits, list(range(1, R + 1)), 0.07, 16)
    ref_scores = oracle.score_columns(logits, list(range(1, R + 1)), [1, R])
    s_k = np.sort(ref_scores)[::-1][k - 1]
    band = 2e-3 * max(abs(s_k), 1.0)
    assert len(got) == len(want) == k
    assert set(np.nonzero(ref_scores > s_k + band)[0]) <= set(got.tolist())
    assert set(got.tolist()) <= set(np.nonzero(ref_scores >= s_k - band)[0])
