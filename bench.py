#!/usr/bin/env python
"""bench.py — one speculation iteration of attention (SURVEY.md §8d unit of work) per step:
per layer verify (gamma+1 rows over the full KV, fused Collect-2 score byproduct, fused append) ->
top-k select (side stream) ; then gamma dependent sparse draft steps over all layers (fused
append).  Metric (BASELINE.json): draft+verify attention tokens/s at 32K ctx = B*(2*gamma+1)/t_iter,
with achieved HBM GB/s against ~8 TB/s and against the measured copy peak.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload config2] [--impl ours|reference]

N > 1 runs under torchrun: one process per GPU, batch-sharded (weak scaling, no data-path
collective in per-layer mode on batch shards), max-over-ranks device time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "draft+verify attention tokens/s at 32K ctx; achieved HBM GB/s vs ~8 TB/s"
HBM_NOMINAL = 8000.0  # GB/s, BASELINE.json denominator

WORKLOADS = {
    # name: (layers, Hq, Hkv, ctx, gamma, batch_per_gpu, description)
    "config2": (32, 32, 8, 32768, 4, 1,
                "Llama-3.1-8B-shaped attention (32q/8kv, d128, 32 layers), 32K ctx, gamma 4, "
                "k=selection_k(0.07,p,16)=2294, batch 1 per GPU"),
    "config1": (1, 32, 8, 4096, 4, 1, "single-layer synthetic, 8 KV heads, d128, 4K ctx, gamma 4"),
    "config3": (32, 32, 8, 65536, 6, 16, "Llama-3.1-8B-shaped, 64K ctx, gamma 6, batch 16 (sharded by batch)"),
    "config4": (80, 64, 8, 131072, 4, 4, "Llama-3.1-70B-shaped (64q/8kv, 80 layers), 128K ctx, gamma 4, batch 4"),
}
RATIO, K_MIN, D = 0.07, 16, 128
STRATEGIES = {"collect2": 4, "all_draft": 3, "last_accepted": 2, "collect2_weights": 5, "quest": 1, "window": 0}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), float(pk.get("bf16_tflops", 1623.5)), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def selection_k(ratio, p, k_min):
    return min(p, max(int(math.floor(ratio * p + 0.5)), k_min))


def iteration_bytes(L, Hq, Hkv, p, gamma, k, B):
    """Algorithmic HBM bytes of one iteration, bf16 KV (s = 2)."""
    s, d = 2, D
    per = ((p + gamma + 1) * 2 * Hkv * d * s                              # verify KV (+ window)
           + sum((k + t) * 2 * Hkv * d * s for t in range(1, gamma + 1))  # draft gathers
           + p * 8 * 2                                                    # per-layer score sums (int64) write + read
           + (gamma + 1) * Hq * d * (s + 4) + gamma * Hq * d * (s + 4)    # Q in (bf16), O out (f32)
           + (gamma + 1) * k * 4                                          # index write + reads
           + (2 * gamma + 1) * 2 * Hkv * d * s)                           # appends
    return per * L * B


def verify_launch_bytes(Hq, Hkv, p, R, B):
    """Algorithmic bytes of ONE verify launch (one layer): KV prefix + window rows + Q + O +
    score byproduct + fused append."""
    d = D
    return B * (p * 2 * Hkv * d * 2 + R * 2 * Hkv * d * 2 + R * Hq * d * 2 + R * Hq * d * 4 + p * 8
                + R * 2 * Hkv * d * 2)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.samples, self._stop = index, [], threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.samples.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 5 + i and s[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# --------------------------------------------------------------------------------------------- ours

def run_ours(args, rank, world, local_rank):
    import torch

    from paper_2602_07223_b200 import COLLECT2, PER_LAYER, Cache, Comm, Runner
    from paper_2602_07223_b200.shard import head_group_ranks, plan
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    L, Hq_full, Hkv_full, ctx, gamma, B_total, desc = WORKLOADS[args.workload]
    if args.gamma:  # config 5: gamma sweep at the workload's context
        gamma = args.gamma
    G = Hq_full // Hkv_full
    strong = args.workload in ("config3", "config4")
    if strong:  # fixed global batch: batch x KV-head shards, shard.plan
        sh = plan(B_total, Hkv_full, world, rank)
        B, Hkv = len(sh.seqs), len(sh.heads)
        seqs_global = B_total
    else:  # config2 / config1: one batch-1 replica per GPU (weak scaling, no collective)
        sh = None
        B, Hkv = B_total, Hkv_full
        seqs_global = B_total * world
    Hq = G * Hkv
    R = gamma + 1
    p0 = ctx
    ratio, k_min = (1e-9, args.k) if args.k else (RATIO, K_MIN)  # config 5: fixed budget k (ratio must be > 0)
    k = selection_k(ratio, p0, k_min)
    scale = 1.0 / math.sqrt(D)
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)

    cache = Cache(L, Hkv, D, p0 + R + 64, max_seqs=B, page_size=256)
    strategy = STRATEGIES[args.strategy]
    # fill the prefix with synthetic post-RoPE keys/values (bf16), chunked appends
    chunk = 2048
    for b in range(B):
        done = 0
        while done < p0:
            n = min(chunk, p0 - done)
            kk = torch.randn((n, L * Hkv, D), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
            vv = torch.randn((n, L * Hkv, D), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
            cache.append(kk, vv, seq=b)
            done += n
    if args.strategy == "quest":
        cache.enable_page_summaries(8)  # SelectorConfig::page_size default (selection.hpp:36)
    torch.cuda.synchronize()
    runner = Runner(cache, Hq, max_rows=R, max_prefix=p0, max_batch=B, sparse_ratio=ratio, k_min=k_min)
    runner.set_batch(list(range(B)), [p0] * B)
    comm = None
    if sh is not None and sh.needs_score_exchange:  # KV heads of a layer on several GPUs: NCCL exchange
        import torch.distributed as dist
        groups = {}
        for base in range(0, world, sh.head_group):  # every rank creates every group (collective call)
            ranks = list(range(base, base + sh.head_group))
            groups[base] = (ranks, dist.new_group(ranks=ranks))
        ranks, grp = groups[head_group_ranks(sh)[0]]
        obj = [Comm.unique_id() if rank == ranks[0] else None]
        dist.broadcast_object_list(obj, src=ranks[0], group=grp)
        comm = Comm(obj[0], len(ranks), ranks.index(rank))
        runner.set_comm(comm)

    def rnd(*shape):
        return torch.randn(shape, generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)

    qv, kvn, vvn = rnd(L, B, Hq, R, D), rnd(L, B, R, Hkv, D), rnd(L, B, R, Hkv, D)
    qd, kdn, vdn = rnd(gamma, L, B, Hq, D), rnd(gamma, L, B, Hkv, D), rnd(gamma, L, B, Hkv, D)
    out_v = torch.empty((L, B, Hq, R, D), dtype=torch.float32, device=dev)
    out_d = torch.empty((gamma, L, B, Hq, D), dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(device=dev)
    itargs = runner.iteration_args(gamma, qv, kvn, vvn, qd, kdn, vdn, out_v, out_d, strategy=strategy,
                                   mode=PER_LAYER, scale=scale, use_graph=not args.no_graph)
    launches_per_step = runner.iteration_kernel_count(itargs)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident timing (inputs already in HBM)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            runner.iteration(itargs, stream=stream)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            runner.iteration(itargs, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    barrier()
    ms = max_over_ranks(ms)

    # ---- dominant kernel (verify): its average duration INSIDE the iteration's PDL chain = the
    # verify-only phase of the same graph (CUDA events on the launching stream) / L launches; the
    # isolated back-to-back launch time is reported beside it
    from paper_2602_07223_b200 import PHASE_DRAFT, PHASE_VERIFY

    def phase_ms(phases, n):
        a = runner.iteration_args(gamma, qv, kvn, vvn, qd, kdn, vdn, out_v, out_d, strategy=strategy, mode=PER_LAYER,
                                  scale=scale, use_graph=not args.no_graph, phases=phases)
        with torch.cuda.stream(stream):
            for _ in range(2):
                runner.iteration(a, stream=stream)
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a0.record(stream)
            for _ in range(n):
                runner.iteration(a, stream=stream)
            a1.record(stream)
        torch.cuda.synchronize()
        return a0.elapsed_time(a1) / n

    v_phase_ms = phase_ms(PHASE_VERIFY, args.steps)
    d_phase_ms = phase_ms(PHASE_DRAFT, args.steps)  # selections of the last full iteration
    with torch.cuda.stream(stream):  # restore a consistent state (sums consumed) for the e2e leg
        runner.iteration(itargs, stream=stream)
    vms = v_phase_ms / L
    nv = min(L, 32)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nv * 3)]
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for i, (a, b_) in enumerate(ev):
            l = i % nv
            a.record(stream)
            runner.verify(l, qv[l], out_v[l], kvn[l], vvn[l], scale, score_row_mask=1 | (1 << gamma), stream=stream)
            b_.record(stream)
            runner.select(l, stream=stream)  # consumes (re-arms) the per-layer score sums, outside the events
    torch.cuda.synchronize()
    vms_isolated = sum(a.elapsed_time(b_) for a, b_ in ev[nv:]) / (len(ev) - nv)  # skip the first (warm) pass

    # ---- end to end through the public API with host buffers (pinned), copies inside the region:
    # every step copies its inputs host->device and reads its outputs back device->host.  Two device
    # buffer sets (two captured graphs) pipeline the transfers: step i+1's inputs go up and step i-1's
    # outputs come down (copy streams, both directions at once) while step i computes.
    dev_sets = [[qv, kvn, vvn, qd, kdn, vdn, out_v, out_d],
                [torch.empty_like(t) for t in (qv, kvn, vvn, qd, kdn, vdn, out_v, out_d)]]
    set_args = [runner.iteration_args(gamma, *d[:6], d[6], d[7], strategy=strategy, mode=PER_LAYER, scale=scale,
                                      use_graph=not args.no_graph) for d in dev_sets]
    n_e2e = args.steps + max(2, args.warmup // 2)  # warm-up covers both buffer sets (both graphs captured)
    host_in = [[t.cpu().pin_memory() for t in (qv, kvn, vvn, qd, kdn, vdn)] for _ in range(2)]
    host_out = [[torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in (out_v, out_d)] for _ in range(2)]
    h2d = sum(t.numel() * t.element_size() for t in host_in[0])
    d2h = sum(t.numel() * t.element_size() for t in host_out[0])
    up, down = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    ev_in = [torch.cuda.Event() for _ in range(n_e2e)]
    ev_done = [torch.cuda.Event() for _ in range(n_e2e)]
    ev_out = [torch.cuda.Event() for _ in range(n_e2e)]

    def upload(i):  # inputs of step i into set i % 2 once step i-2 (same set) is computed AND read back
        st = i % 2
        if i >= 2:
            up.wait_event(ev_out[i - 2])  # implies ev_done[i - 2]; the compute stream then waits on ev_in only
        with torch.cuda.stream(up):
            for h, d_ in zip(host_in[st], dev_sets[st][:6]):
                d_.copy_(h, non_blocking=True)
        ev_in[i].record(up)

    def e2e_run(lo, hi):
        upload(lo)
        for i in range(lo, hi):
            st = i % 2
            if i + 1 < hi:
                upload(i + 1)
            stream.wait_event(ev_in[i])  # (ev_in[i] follows ev_out[i - 2]: set st's outputs are free)
            runner.iteration(set_args[st], stream=stream)
            ev_done[i].record(stream)
            down.wait_event(ev_done[i])
            with torch.cuda.stream(down):
                for h, d_ in zip(host_out[st], dev_sets[st][6:]):
                    h.copy_(d_, non_blocking=True)
            ev_out[i].record(down)

    e2e_run(0, n_e2e - args.steps)  # warm-up (captures the second graph)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_start.record(up)  # the region opens before the first upload ...
    e2e_run(n_e2e - args.steps, n_e2e)
    stream.wait_event(ev_out[n_e2e - 1])
    t_end.record(stream)  # ... and closes after the last read-back
    torch.cuda.synchronize()
    ms_e2e = max_over_ranks(t_start.elapsed_time(t_end) / args.steps)

    hbm_peak, _, peak_src = peaks()
    tok_per_step = seqs_global * (2 * gamma + 1)  # whole job: every sequence counted once
    value = tok_per_step / (ms / 1e3)
    it_bytes = iteration_bytes(L, Hq, Hkv, p0, gamma, k, B)
    vb = verify_launch_bytes(Hq, Hkv, p0, R, B)
    v_gbs = vb / (vms / 1e3) / 1e9
    draft_bytes = B * ((k + (gamma + 1) / 2) * 2 * Hkv * D * 2 + Hq * D * 6 + k * 4 + 2 * Hkv * D * 2)
    traffic = None
    tf = os.path.join(ROOT, "profiles", "verify_dram_bytes.json")  # ncu dram__bytes_{read,write}.sum per launch
    if os.path.exists(tf):
        try:
            with open(tf) as f:
                t = json.load(f)
            if t.get("workload") == args.workload:
                traffic = t.get("bytes_per_launch")
        except Exception:
            traffic = None
    it_gbs = it_bytes / (ms / 1e3) / 1e9
    result = {
        "metric": METRIC, "value": round(value, 2), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (torch.randn, post-RoPE K/V/Q, bf16)",
        "config": {"workload": (f"config5 sweep point (gamma {gamma}, k {k}) on {args.workload}'s shape"
                                if args.gamma or args.k else f"{args.workload}: {desc}"),
                   "global_batch": seqs_global, "seq_len": p0,
                   "gamma": gamma, "k": k, "selection": f"{args.strategy}, per-layer", "layers": L,
                   "parallelism": (f"{world} GPUs: batch x KV-head shards ({B} seq x {Hkv} KV heads per GPU"
                                   + (f", NCCL per-layer score exchange over {sh.head_group} GPUs)" if comm else ")")
                                   if strong else f"dp{world} (one batch-1 replica per GPU, no collective)"),
                   "l2": f"inputs > L2: KV cache {L * B * p0 * Hkv * D * 4 / 1e9:.1f} GB/GPU >> 126 MB",
                   "cuda_graph": not args.no_graph},
        "hbm": {"per_gpu": True, "bytes_per_iter": it_bytes, "achieved_gbs": round(it_gbs, 1),
                "frac_of_8tbs": round(it_gbs / HBM_NOMINAL, 4), "frac_of_measured": round(it_gbs / hbm_peak, 4),
                "measured_peak_gbs": hbm_peak, "peak_source": peak_src},
        "roofline": {"kernel": "verify_tc_kernel (one layer, all KV heads)", "bound": "hbm", "achieved": round(v_gbs, 1),
                     "peak": hbm_peak, "unit": "GB/s", "frac": round(v_gbs / hbm_peak, 4), "traffic": traffic,
                     "bytes_per_launch": vb, "launch_us": round(vms * 1e3, 2),
                     "launch_us_isolated": round(vms_isolated * 1e3, 2), "peak_source": peak_src,
                     "timing": "verify-only phase of the iteration graph (PDL chain, CUDA events) / L launches"},
        "phases": {"verify_ms": round(v_phase_ms, 4), "draft_ms": round(d_phase_ms, 4),
                   "draft_us_per_launch": round(d_phase_ms * 1e3 / (gamma * L), 2),
                   "draft_bytes_per_launch": draft_bytes, "draft_gbs": round(draft_bytes / (d_phase_ms / (gamma * L) / 1e3) / 1e9, 1)},
        "e2e": {"value": round(tok_per_step / (ms_e2e / 1e3), 2), "unit": "tokens/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": round(ms_e2e, 4),
                "how": "public API (sa_iteration_run graph), pinned host inputs/outputs copied every step; "
                       "two buffer sets pipeline step i+1's upload and step i-1's read-back with step i"},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_extras:
        result["next_rows"] = next_rows(dev, B, gamma, hbm_peak)
    return result


def next_rows(dev, B, gamma, hbm_peak):
    """SURVEY.md §8f rows measured beside the headline (not part of `value`): the model-side producer
    (RMSNorm + fused QKV projection + RoPE, Llama-3.1-8B shape, a 32-layer PDL chain in one graph) for
    the verify rows and a draft row, and the speculation acceptance kernel at the Llama-3 vocabulary."""
    import torch

    from paper_2602_07223_b200 import QkvProjection, accept
    L, Dm, Hq, Hkv = 32, 4096, 32, 8
    n_out = (Hq + 2 * Hkv) * 128
    g = torch.Generator(device=dev)
    g.manual_seed(99)
    w = (torch.randn((L, n_out, Dm), generator=g, device=dev) / 64).to(torch.bfloat16)
    proj = QkvProjection(w, torch.ones((L, Dm), device=dev), Hq, Hkv)
    del w
    out = {}
    s = torch.cuda.Stream(device=dev)
    for name, rows in (("verify_rows", gamma + 1), ("draft_row", 1)):
        x = torch.randn((B, rows, Dm), generator=g, device=dev)
        pos = torch.full((B,), 32768, dtype=torch.int32, device=dev)
        q = torch.empty((B, Hq, rows, 128), dtype=torch.bfloat16, device=dev)
        kn = torch.empty((B, rows, Hkv, 128), dtype=torch.bfloat16, device=dev)
        vn = torch.empty_like(kn)
        with torch.cuda.stream(s):
            for l in range(L):
                proj.project(l, x, pos, q, kn, vn, stream=s)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                for l in range(L):
                    proj.project(l, x, pos, q, kn, vn, stream=s)
            for _ in range(3):
                gr.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(10):
                gr.replay()
            e1.record(s)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (10 * L)
        nbytes = n_out * Dm * 2 + B * rows * (Dm * 4 + n_out * 2)
        gbs = nbytes / us / 1e3
        out[name] = {"tokens": B * rows, "us_per_layer": round(us, 2), "bytes_per_layer": nbytes,
                     "achieved_gbs": round(gbs, 1), "frac": round(gbs / hbm_peak, 4)}
    proj.close()
    res = {"producer": dict(out, kernel="qkv_gemv (one fused mma.sync launch: RMSNorm + QKV + RoPE, <= 8 tokens)", shape="Llama-3.1-8B layer",
                            chain="32 layers, one CUDA graph, PDL")}
    V = 128256
    p = torch.softmax(torch.randn((B, gamma + 1, V), generator=g, device=dev), -1)
    qd = torch.softmax(torch.randn((B, gamma, V), generator=g, device=dev), -1)
    draft = torch.randint(0, V, (B, gamma), generator=g, device=dev, dtype=torch.int32)
    u = torch.rand((B, gamma + 1), generator=g, device=dev)
    res_out = (torch.empty(B, dtype=torch.int32, device=dev), torch.empty((B, gamma + 1), dtype=torch.int32, device=dev))
    with torch.cuda.stream(s):  # a graph of 20 calls: device time, not Python launch overhead
        accept(p, draft, q=qd, u=u, stream=s, out=res_out)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            for _ in range(20):
                accept(p, draft, q=qd, u=u, stream=s, out=res_out)
        gr.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        gr.replay()
        e1.record(s)
    torch.cuda.synchronize()
    res["accept"] = {"us_per_call": round(e0.elapsed_time(e1) * 1e3 / 20, 2), "vocab": V, "gamma": gamma, "batch": B,
                     "mode": "modified rejection sampling"}
    # the CPU restatements timed beside them (host cores of this box; the reference ships no code here)
    import numpy as np

    from oracle.model import qkv_project
    from oracle.speculation import accept as ref_accept
    rng = np.random.default_rng(3)
    wn = rng.standard_normal((n_out, Dm)).astype(np.float32)
    xn = rng.standard_normal((B, gamma + 1, Dm)).astype(np.float32)
    t0 = time.perf_counter()
    qkv_project(xn, wn, np.ones(Dm, np.float32), Hq, Hkv, [32768] * B)
    res["producer"]["cpu_port"] = {"us_per_layer": round((time.perf_counter() - t0) * 1e6, 1),
                                   "kind": "port (oracle/model.py, numpy float64)", "tokens": B * (gamma + 1),
                                   "cores": os.cpu_count()}
    pn, qn = p[0].cpu().numpy(), qd[0].cpu().numpy()
    t0 = time.perf_counter()
    ref_accept(pn, draft[0].cpu().numpy(), q=qn, u=u[0].cpu().numpy())
    res["accept"]["cpu_port"] = {"us_per_call": round((time.perf_counter() - t0) * 1e6, 1),
                                 "kind": "port (oracle/speculation.py, scalar Python)", "batch": 1, "cores": 1}
    return res


# --------------------------------------------------------------------------------------------- CPU

class CpuReferenceSample:
    """Reference CPU path (oracle/_ref = the reference's own TUs) on a bounded sample of the workload:
    one layer (verify of all q-heads x rows over the full prefix, Collect-2 select, gamma draft steps),
    extrapolated x layers.  The prefix is appended once; every step() re-runs the sample on it."""

    def __init__(self, workload, threads):
        import numpy as np

        from oracle.pyoracle import REF_SO, Oracle, Ref
        self.L, self.Hq, self.Hkv, self.ctx, self.gamma, self.B, _ = WORKLOADS[workload]
        self.workload = workload
        self.kind = "reference"
        try:
            impl = Ref() if os.path.exists(REF_SO) else None
        except Exception:
            impl = None
        if impl is None:
            impl, self.kind, threads = Oracle(), "port", 1
        self.impl, self.threads = impl, threads
        p0, R = self.ctx, self.gamma + 1
        self.rng = np.random.default_rng(7)
        self.kv = impl.kv(1, self.Hkv, D, p0 + R + 8)
        self.K = self.rng.standard_normal((p0 + R, self.Hkv, D), dtype=np.float32)
        self.V = self.rng.standard_normal((p0 + R, self.Hkv, D), dtype=np.float32)
        for t in range(p0):
            self.kv.append(self.K[t], self.V[t])
        self.q = self.rng.standard_normal((self.Hq, R, D), dtype=np.float32)

    def step(self):
        """One sample; returns (tokens/s extrapolated to the workload, seconds, description)."""
        import numpy as np

        from oracle.pyoracle import COLLECT2
        p0, R, gamma, L, B = self.ctx, self.gamma + 1, self.gamma, self.L, self.B
        scale = 1.0 / math.sqrt(D)
        kwargs = {"threads": self.threads} if self.kind == "reference" else {}
        self.kv.truncate(p0)
        for t in range(R):  # the gamma+1 verify rows
            self.kv.append(self.K[p0 + t], self.V[p0 + t])
        t0 = time.perf_counter()
        _, logits = self.kv.verify_layer(0, self.Hq, self.q, p0, R, scale, **kwargs)
        t1 = time.perf_counter()
        sel = self.impl.select(COLLECT2, logits, list(range(1, R + 1)), RATIO, K_MIN)
        t2 = time.perf_counter()
        self.kv.truncate(p0)
        for j in range(1, gamma + 1):
            self.kv.append(self.K[p0 + j - 1], self.V[p0 + j - 1])
            self.kv.draft_layer(0, self.Hq, self.rng.standard_normal((self.Hq, D), dtype=np.float32), [sel], p0, j,
                                scale, **kwargs)
        t3 = time.perf_counter()
        per_layer = t3 - t0
        tps = B * (2 * gamma + 1) / (per_layer * L * B)
        sample = (f"1 of {L} layers x batch 1 of {B} ({self.workload}): verify {self.Hq}x{R} attend_collect over "
                  f"{p0} keys {t1 - t0:.2f}s + collect2 select {t2 - t1:.2f}s + {gamma} draft steps {t3 - t2:.2f}s; "
                  f"extrapolated x{L * B}")
        return tps, per_layer, sample


def cpu_reference_sample(workload, threads):
    """One bounded, warm sample of the reference CPU path (after one untimed sample):
    (tokens/s, seconds, description, kind)."""
    ref = CpuReferenceSample(workload, threads)
    ref.step()
    tps, secs, sample = ref.step()
    return tps, secs, sample, ref.kind


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation (oracle/_ref), all host threads, W
    untimed samples then K timed ones (each sample one layer of the workload, extrapolated)."""
    if rank != 0:
        return None
    threads = os.cpu_count() or 1
    ref = CpuReferenceSample(args.workload, threads)
    for _ in range(args.warmup):
        ref.step()
    secs, sample = 0.0, ""
    for _ in range(args.steps):
        _, s1, sample = ref.step()
        secs += s1
    L, Hq, Hkv, ctx, gamma, B, desc = WORKLOADS[args.workload]
    v = args.steps * B * (2 * gamma + 1) / (secs * L * B)  # K samples, each one layer of L
    cores = threads if ref.kind == "reference" else 1
    return {
        "metric": METRIC, "value": round(v, 4), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * B * (2 * gamma + 1) / v, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64 (reference CPU arithmetic)",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": f"{args.workload}: {desc}", "global_batch": B, "seq_len": ctx, "gamma": gamma},
        "cpu_baseline": {"value": round(v, 4), "unit": "tokens/s", "cores": cores, "kind": ref.kind,
                         "sample": f"each step: {sample}"},
        "e2e": {"value": round(v, 4), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="config2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--gamma", type=int, default=0, help="override the workload's gamma (config 5 sweep)")
    ap.add_argument("--k", type=int, default=0, help="fixed selection budget k instead of selection_k(0.07, p, 16)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the §8f next-row measurements")
    ap.add_argument("--strategy", default="collect2", choices=sorted(STRATEGIES),
                    help="selection strategy of the iteration (the headline is collect2; the others are the "
                         "paper's variants / baselines for the overhead comparison)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        res = run_reference(args, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    res = run_ours(args, rank, world, local_rank)
    if rank == 0:
        if not args.no_cpu_baseline:
            try:
                tps, _, sample, kind = cpu_reference_sample(args.workload, os.cpu_count() or 1)
                res["cpu_baseline"] = {"value": round(tps, 4), "unit": "tokens/s",
                                       "cores": (os.cpu_count() or 1) if kind == "reference" else 1,
                                       "kind": kind, "sample": sample}
            except Exception as e:  # reported, never fatal
                res["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
