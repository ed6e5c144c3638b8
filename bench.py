#!/usr/bin/env python
"""bench.py — one speculation iteration of attention (SURVEY.md §8d unit of work) per step:
per layer verify (gamma+1 rows over the full KV, fused Collect-2 score byproduct, fused append) ->
top-k select (side stream) ; then gamma dependent sparse draft steps over all layers (fused
append).  Metric (BASELINE.json): draft+verify attention tokens/s at 32K ctx = B*(2*gamma+1)/t_iter,
with achieved HBM GB/s against ~8 TB/s and against the measured copy peak.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload configX] [--impl ours|reference]
                  [--data gaussian|structured] [--shard replica|plan|heads]

--gpus N > 1 starts its own N ranks (torch.distributed.run, one process per GPU) unless it already
runs under torchrun.  N = 1 defaults to config2 (the BASELINE metric's config); N > 1 defaults to
config3 (B = 16 sharded batch-first, then KV heads: strong scaling) and adds a "headsplit" run of the
config-4 shape with its KV heads split over all N GPUs, where every layer's per-layer selection
exchanges the int64 column sums over NCCL inside the iteration graph.  Device time is the max over
ranks; `value` counts every sequence of the job once.
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
if os.environ.get("SA_AB_ROOT"):  # dev A/B runs (tools/ab_build.sh): the package from another build
    sys.path.insert(0, os.path.abspath(os.environ["SA_AB_ROOT"]))

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


def iteration_bytes(L, Hq, Hkv, p, gamma, k, B, accepted=None):
    """Algorithmic HBM bytes of one iteration, bf16 KV (s = 2).  The draft phase is the
    next draft chain after accepting `accepted` drafts (default gamma): step t reads T plus the tail
    [p, p + accepted + 1 + t)."""
    s, d = 2, D
    a1 = (gamma if accepted is None else accepted) + 1
    per = ((p + gamma + 1) * 2 * Hkv * d * s                              # verify KV (+ window)
           + sum((k + a1 + t) * 2 * Hkv * d * s for t in range(1, gamma + 1))  # draft gathers
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

def shard_for(workload, mode, world, rank):
    """(shard or None, B local, Hkv local, sequences counted once over the whole job, strong?)."""
    from paper_2602_07223_b200.shard import plan, plan_heads
    L, Hq, Hkv, ctx, gamma, B_total, _ = WORKLOADS[workload]
    if mode == "replica":  # one full copy of the workload per GPU (weak scaling, no collective)
        return None, B_total, Hkv, B_total * world, False
    sh = (plan if mode == "plan" else plan_heads)(B_total, Hkv, world, rank)
    return sh, len(sh.seqs), len(sh.heads), B_total, True


def run_ours(args, rank, world, local_rank, workload, mode, data="gaussian", steps=None, warmup=None,
             e2e=True, label=None):
    """One measured configuration: fill the cache, capture the iteration graph, time K iterations on the
    device (max over ranks), then the end-to-end leg through the public API with host buffers."""
    import numpy as np
    import torch

    from paper_2602_07223_b200 import PER_LAYER, Cache, Comm, Runner
    from paper_2602_07223_b200.shard import head_group_ranks
    from paper_2602_07223_b200.synthetic import default_shift, heavy_hitter_positions, plant_shift, plant_torch
    steps = steps or args.steps
    warmup = max(3, warmup or args.warmup)
    local_rank = _local_device(local_rank)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    L, Hq_full, Hkv_full, ctx, gamma, B_total, desc = WORKLOADS[workload]
    if args.gamma:  # config 5: gamma sweep at the workload's context
        gamma = args.gamma
    G = Hq_full // Hkv_full
    emu = getattr(args, "emulate_world", 0) if world == 1 else 0
    # --emulate-world N (one GPU): run rank 0's shard of an N-GPU job; the score exchange runs on a
    # one-rank communicator (its launch in the graph, not the NVLink transfer)
    sh, B, Hkv, seqs_global, strong = shard_for(workload, mode, emu or world, rank)
    Hq = G * Hkv
    R = gamma + 1
    p0 = ctx
    accepted = gamma  # the timing unit's next draft chain starts after all gamma drafts are accepted
    ratio, k_min = (1e-9, args.k) if args.k else (RATIO, K_MIN)  # config 5: fixed budget k (ratio must be > 0)
    k = selection_k(ratio, p0, k_min)
    scale = 1.0 / math.sqrt(D)
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)

    def rnd(*shape):
        return torch.randn(shape, generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)

    # queries first: the structured variant plants its heavy hitters along them
    qv, kvn, vvn = rnd(L, B, Hq, R, D), rnd(L, B, R, Hkv, D), rnd(L, B, R, Hkv, D)
    qd, kdn, vdn = rnd(gamma, L, B, Hq, D), rnd(gamma, L, B, Hkv, D), rnd(gamma, L, B, Hkv, D)
    planted = None
    if data == "structured":
        rng = np.random.default_rng(4321 + rank)
        qc = qv[:, :, :, [0, gamma]].float().cpu().numpy()  # the Collect-2 rows score the columns
        planted, deltas = [], []
        for b in range(B):
            planted.append([heavy_hitter_positions(p0, k, rng) for _ in range(L)])
            deltas.append(torch.from_numpy(np.stack([np.stack([plant_shift(qc[l, b, gg * G:(gg + 1) * G], default_shift())
                                                               for gg in range(Hkv)]) for l in range(L)])).to(dev))

    cache = Cache(L, Hkv, D, p0 + 2 * R + 64, max_seqs=B, page_size=256)
    chunk = 2048
    for b in range(B):  # the prefix: synthetic post-RoPE keys/values (bf16), chunked appends
        done = 0
        while done < p0:
            n = min(chunk, p0 - done)
            kk = torch.randn((n, L * Hkv, D), generator=g, device=dev, dtype=torch.float32)
            if planted is not None:
                plant_torch(kk, done, planted[b], deltas[b])
            vv = torch.randn((n, L * Hkv, D), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
            cache.append(kk.to(torch.bfloat16), vv, seq=b)
            done += n
    if args.strategy == "quest":
        cache.enable_page_summaries(8)  # SelectorConfig::page_size default (selection.hpp:36)
    torch.cuda.synchronize()
    runner = Runner(cache, Hq, max_rows=R, max_prefix=p0, max_batch=B, sparse_ratio=ratio, k_min=k_min)
    for kv_ in args.dev:  # dev-only knobs (sa_dev_set_knob), e.g. --dev iter_skip=6
        name, val = kv_.split("=")
        runner.set_dev_knob(name, int(val))
    runner.set_batch(list(range(B)), [p0] * B)
    comm, comm_info = None, None
    if sh is not None and sh.needs_score_exchange and emu:
        comm = Comm(Comm.unique_id(), 1, 0)
        comm_info = {"nranks": 1, "rank": 0, "group": [0], "ok": True,
                     "emulated": f"rank 0 of a {emu}-GPU head group; one-rank communicator"}
        runner.set_comm(comm)
    elif sh is not None and sh.needs_score_exchange:  # KV heads of a layer on several GPUs: NCCL exchange
        import torch.distributed as dist
        groups = {}
        for base in range(0, world, sh.head_group):  # every rank creates every group (collective call)
            ranks = list(range(base, base + sh.head_group))
            groups[base] = (ranks, dist.new_group(ranks=ranks))
        ranks, grp = groups[head_group_ranks(sh)[0]]
        obj = [Comm.unique_id() if rank == ranks[0] else None]
        dist.broadcast_object_list(obj, src=ranks[0], group=grp)
        comm = Comm(obj[0], len(ranks), ranks.index(rank))
        n_nccl, r_nccl = comm.info()
        comm_info = {"nranks": n_nccl, "rank": r_nccl, "group": ranks, "ok": n_nccl == len(ranks)}
        print(f"[rank {rank}] NCCL score-exchange communicator: {n_nccl} ranks (group {ranks}), rank {r_nccl}",
              file=sys.stderr, flush=True)
        runner.set_comm(comm)

    strategy = STRATEGIES[args.strategy]
    out_v = torch.empty((L, B, Hq, R, D), dtype=torch.float32, device=dev)
    out_d = torch.empty((gamma, L, B, Hq, D), dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(device=dev)

    def it_args(bufs=(qv, kvn, vvn, qd, kdn, vdn, out_v, out_d), phases=0):
        return runner.iteration_args(gamma, *bufs, strategy=strategy, mode=(1 if args.per_kv_head else PER_LAYER),
                                     scale=scale,
                                     use_graph=not args.no_graph, phases=phases, accepted=accepted)

    itargs = it_args()
    launches_per_step = runner.iteration_kernel_count(itargs)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if _SHARED_GPU else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sync():
        if comm is not None:
            comm.sync(stream, timeout_ms=600000)  # watches NCCL: a dead peer aborts instead of hanging
        torch.cuda.synchronize()

    # ---- device-resident timing (inputs already in HBM; the KV cache is >> L2)
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            runner.iteration(itargs, stream=stream)
    sync()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        for _ in range(steps):
            runner.iteration(itargs, stream=stream)
        e1.record(stream)
        sync()
    ms = e0.elapsed_time(e1) / steps
    barrier()
    ms = max_over_ranks(ms)

    # recall of the planted heavy hitters by the selections of the last iteration (structured data)
    recall = None
    if planted is not None:
        hit = tot = 0
        for layer in range(L):
            idx, cnt = runner.selection(layer, 1)
            for b in range(B):
                got = set(idx[b, 0, : cnt[b, 0]].tolist())
                hit += sum(1 for x in planted[b][layer].tolist() if x in got)
                tot += len(planted[b][layer])
        recall = hit / max(tot, 1)

    # ---- phase split inside the same graph structure (CUDA events on the launching stream): the
    # draft phase alone (selections of the last full iteration), so the verify chain's share of the
    # FULL iteration (selects running on the side stream) is ms - draft; and the verify-only phase
    from paper_2602_07223_b200 import PHASE_DRAFT, PHASE_VERIFY

    def phase_ms(phases, n):
        a = it_args(phases=phases)
        with torch.cuda.stream(stream):
            for _ in range(2):
                runner.iteration(a, stream=stream)
        sync()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a0.record(stream)
            for _ in range(n):
                runner.iteration(a, stream=stream)
            a1.record(stream)
        sync()
        return max_over_ranks(a0.elapsed_time(a1) / n)

    v_only_ms = phase_ms(PHASE_VERIFY, steps)
    d_phase_ms = phase_ms(PHASE_DRAFT, steps)
    with torch.cuda.stream(stream):  # restore a consistent state (sums consumed) for the e2e leg
        runner.iteration(itargs, stream=stream)
    sync()
    v_in_iter_ms = max(ms - d_phase_ms, 1e-9)  # verify chain (+ overlapped selects) inside the iteration

    # ---- end to end through the public API with host buffers (pinned), copies inside the region:
    # every step copies its inputs host->device and reads its outputs back device->host.  Three device
    # buffer sets (three captured graphs) pipeline the transfers: step i+1's inputs go up and step i-1's
    # outputs come down (copy streams, both directions at once) while step i computes (two sets measured
    # 0.1-0.3 % slower: the upload of step i+1 then waits for the read-back of step i-1).
    e2e_res = None
    if e2e:
        NS = int(os.environ.get("SA_E2E_SETS", 3))  # device buffer sets in flight (dev A/B knob)
        dev_sets = [[qv, kvn, vvn, qd, kdn, vdn, out_v, out_d]] + \
                   [[torch.empty_like(t) for t in (qv, kvn, vvn, qd, kdn, vdn, out_v, out_d)] for _ in range(NS - 1)]
        set_args = [it_args(tuple(d)) for d in dev_sets]
        n_e2e = steps + max(NS, warmup // 2)  # warm-up covers every buffer set (every graph captured)
        host_in = [[t.cpu().pin_memory() for t in (qv, kvn, vvn, qd, kdn, vdn)] for _ in range(NS)]
        host_out = [[torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in (out_v, out_d)] for _ in range(NS)]
        h2d = sum(t.numel() * t.element_size() for t in host_in[0])
        d2h = sum(t.numel() * t.element_size() for t in host_out[0])
        up, down = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        ev_in = [torch.cuda.Event() for _ in range(n_e2e)]
        ev_done = [torch.cuda.Event() for _ in range(n_e2e)]
        ev_out = [torch.cuda.Event() for _ in range(n_e2e)]

        def upload(i):  # inputs of step i into set i % NS once step i-NS (same set) is computed AND read back
            st = i % NS
            if i >= NS:
                up.wait_event(ev_out[i - NS])  # implies ev_done[i - NS]; the compute stream then waits on ev_in only
            with torch.cuda.stream(up):
                for h, d_ in zip(host_in[st], dev_sets[st][:6]):
                    d_.copy_(h, non_blocking=True)
            ev_in[i].record(up)

        def e2e_run(lo, hi):
            upload(lo)
            for i in range(lo, hi):
                st = i % NS
                if i + 1 < hi:
                    upload(i + 1)
                stream.wait_event(ev_in[i])  # (ev_in[i] follows ev_out[i - NS]: set st's outputs are free)
                runner.iteration(set_args[st], stream=stream)
                ev_done[i].record(stream)
                down.wait_event(ev_done[i])
                with torch.cuda.stream(down):
                    for h, d_ in zip(host_out[st], dev_sets[st][6:]):
                        h.copy_(d_, non_blocking=True)
                ev_out[i].record(down)

        e2e_run(0, n_e2e - steps)  # warm-up (captures the second graph)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t_start.record(up)  # the region opens before the first upload ...
        e2e_run(n_e2e - steps, n_e2e)
        stream.wait_event(ev_out[n_e2e - 1])
        t_end.record(stream)  # ... and closes after the last read-back
        sync()
        ms_e2e = max_over_ranks(t_start.elapsed_time(t_end) / steps)
        tok_per_step = seqs_global * (2 * gamma + 1)
        e2e_res = {"value": round(tok_per_step / (ms_e2e / 1e3), 2), "unit": "tokens/s",
                   "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": round(ms_e2e, 4),
                   "how": "public API (sa_iteration_run graph), pinned host inputs/outputs copied every step; "
                          "three buffer sets pipeline step i+1's upload and step i-1's read-back with step i"}
    if comm is not None:
        comm.check()

    hbm_peak, _, peak_src = peaks()
    tok_per_step = seqs_global * (2 * gamma + 1)  # whole job: every sequence counted once
    value = tok_per_step / (ms / 1e3)
    it_bytes = iteration_bytes(L, Hq, Hkv, p0, gamma, k, B, accepted)
    vb = verify_launch_bytes(Hq, Hkv, p0, R, B)
    v_gbs = vb / (v_in_iter_ms / L / 1e3) / 1e9
    v_only_gbs = vb / (v_only_ms / L / 1e3) / 1e9
    draft_bytes = B * ((k + accepted + 1 + (gamma + 1) / 2) * 2 * Hkv * D * 2 + Hq * D * 6 + k * 4 + 2 * Hkv * D * 2)
    traffic, traffic_src = None, None
    tf = os.path.join(ROOT, "profiles", "verify_dram_bytes.json")  # ncu dram__bytes_{read,write}.sum per launch
    if os.path.exists(tf):
        try:
            with open(tf) as f:
                t = json.load(f)
            if t.get("workload") == workload and t.get("gamma", 4) == gamma:
                traffic, traffic_src = t.get("bytes_per_launch"), t.get("source")
        except Exception:
            traffic = None
    it_gbs = it_bytes / (ms / 1e3) / 1e9
    par = ("dp%d (one batch-%d replica per GPU, no collective)" % (world, B) if sh is None else
           (f"EMULATED rank 0 of {emu}: " if emu else "") +
           f"{emu or world} GPUs: batch x KV-head shards ({B} seq x {Hkv} KV heads per GPU"
           + (f", NCCL per-layer score exchange over {sh.head_group} GPUs)" if comm else ", no collective)"))
    result = {
        "metric": METRIC, "value": round(value, 2), "unit": "tokens/s", "n_gpus": world, "steps": steps,
        "warmup": warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": ("synthetic (torch.randn, post-RoPE K/V/Q, bf16)" if data == "gaussian" else
                 "synthetic structured (torch.randn + planted heavy hitters: k/4 keys per layer shifted along the "
                 "mean Collect-2 query so their mean logit rises by 3*sqrt(d))"),
        "config": {"workload": label or (f"config5 sweep point (gamma {gamma}, k {k}) on {workload}'s shape"
                                         if args.gamma or args.k else f"{workload}: {desc}"),
                   "global_batch": seqs_global, "seq_len": p0,
                   "gamma": gamma, "k": k, "selection": f"{args.strategy}, " + ("per-KV-head" if args.per_kv_head else "per-layer"), "layers": L,
                   "accepted": accepted, "parallelism": par,
                   "l2": f"inputs > L2: KV cache {L * B * p0 * Hkv * D * 4 / 1e9:.1f} GB/GPU >> 126 MB",
                   "cuda_graph": not args.no_graph},
        "hbm": {"per_gpu": True, "bytes_per_iter": it_bytes, "achieved_gbs": round(it_gbs, 1),
                "frac_of_8tbs": round(it_gbs / HBM_NOMINAL, 4), "frac_of_measured": round(it_gbs / hbm_peak, 4),
                "measured_peak_gbs": hbm_peak, "peak_source": peak_src},
        "roofline": {"kernel": "verify_tc_kernel (one layer, all KV heads)", "bound": "hbm", "achieved": round(v_gbs, 1),
                     "peak": hbm_peak, "unit": "GB/s", "frac": round(v_gbs / hbm_peak, 4), "traffic": traffic,
                     "traffic_source": traffic_src, "bytes_per_launch": vb,
                     "launch_us": round(v_in_iter_ms * 1e3 / L, 2),
                     "timing": "inside the full iteration: (iteration - draft phase) / L, CUDA events on the "
                               "launching stream (the selects run beside the verify chain)",
                     "verify_only_launch_us": round(v_only_ms * 1e3 / L, 2),
                     "verify_only_frac": round(v_only_gbs / hbm_peak, 4), "peak_source": peak_src},
        "phases": {"verify_in_iteration_ms": round(v_in_iter_ms, 4), "verify_only_ms": round(v_only_ms, 4),
                   "draft_ms": round(d_phase_ms, 4), "draft_us_per_launch": round(d_phase_ms * 1e3 / (gamma * L), 2),
                   "draft_bytes_per_launch": draft_bytes,
                   "draft_gbs": round(draft_bytes / (d_phase_ms / (gamma * L) / 1e3) / 1e9, 1)},
        "gpu_launches": launches_per_step * steps,
        "clocks": clk.summary(),
    }
    if e2e_res is not None:
        result["e2e"] = e2e_res
    if recall is not None:
        result["heavy_hitter_recall"] = round(recall, 6)
    if comm_info is not None:
        result["comm"] = comm_info
    if emu:
        result["emulated"] = {"world": emu, "note": "one GPU runs rank 0's shard; value = whole-job tokens / "
                              "rank 0's iteration time (every rank's shard is identical); the per-layer score "
                              "all-reduce runs on a one-rank communicator (no NVLink transfer)"}
    if comm is not None:
        runner.set_comm(None)
        comm.close()
    runner.close()
    cache.close()
    del qv, kvn, vvn, qd, kdn, vdn, out_v, out_d
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
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

def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class CpuReferenceSample:
    """Reference CPU path (oracle/_ref = the reference's own TUs) on one sequence of the workload: per
    layer, verify of all q-heads x rows over the full prefix (attend_collect), the Collect-2 select and
    the gamma draft steps (gather + attend) of the next draft chain.  The store holds one layer's KV and
    each 'layer' of a step re-runs that layer's arithmetic on it (the same work as a distinct layer; one
    layer's fp32 KV, 268 MB at 32K, is far larger than any CPU cache)."""

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
        self.kv = impl.kv(1, self.Hkv, D, p0 + 2 * R + 8)
        self.K = self.rng.standard_normal((p0 + 2 * R, self.Hkv, D), dtype=np.float32)
        self.V = self.rng.standard_normal((p0 + 2 * R, self.Hkv, D), dtype=np.float32)
        for t in range(p0):
            self.kv.append(self.K[t], self.V[t])
        self.q = self.rng.standard_normal((self.Hq, R, D), dtype=np.float32)

    def layer(self, threads=None):
        """One layer of one sequence; returns (seconds, (verify, select, drafts) seconds)."""
        import numpy as np

        from oracle.pyoracle import COLLECT2
        p0, R, gamma = self.ctx, self.gamma + 1, self.gamma
        scale = 1.0 / math.sqrt(D)
        kwargs = {"threads": threads or self.threads} if self.kind == "reference" else {}
        self.kv.truncate(p0)
        for t in range(R):  # the gamma+1 verify rows
            self.kv.append(self.K[p0 + t], self.V[p0 + t])
        t0 = time.perf_counter()
        _, logits = self.kv.verify_layer(0, self.Hq, self.q, p0, R, scale, **kwargs)
        t1 = time.perf_counter()
        sel = self.impl.select(COLLECT2, logits, list(range(1, R + 1)), RATIO, K_MIN)
        t2 = time.perf_counter()
        a1 = gamma + 1  # the next draft chain after accepting all gamma drafts (bench's timing unit)
        self.kv.truncate(p0 + a1)
        for j in range(1, gamma + 1):
            self.kv.append(self.K[p0 + a1 + j - 1], self.V[p0 + a1 + j - 1])
            self.kv.draft_layer(0, self.Hq, self.rng.standard_normal((self.Hq, D), dtype=np.float32), [sel], p0,
                                a1 + j, scale, **kwargs)
        t3 = time.perf_counter()
        return t3 - t0, (t1 - t0, t2 - t1, t3 - t2)

    def step(self, n_layers, threads=None):
        """n_layers layers of one sequence: (seconds, phase seconds summed)."""
        tot, ph = 0.0, [0.0, 0.0, 0.0]
        for _ in range(n_layers):
            s, p = self.layer(threads)
            tot += s
            ph = [a + b for a, b in zip(ph, p)]
        return tot, ph


def cpu_baseline(workload):
    """My arm's cpu_baseline: a bounded, warm sample (one layer of one sequence) of the reference CPU path
    on all host threads, extrapolated to the workload, plus the single-threaded figure (the reference
    itself is single-threaded, attention.cpp:38-66)."""
    threads = os.cpu_count() or 1
    ref = CpuReferenceSample(workload, threads)
    L, B, gamma = ref.L, ref.B, ref.gamma
    ref.layer()  # warm
    secs, ph = ref.layer()
    tps = B * (2 * gamma + 1) / (secs * L * B)
    out = {"value": round(tps, 4), "unit": "tokens/s", "cores": threads if ref.kind == "reference" else 1,
           "kind": ref.kind, "cpu": cpu_model(),
           "sample": (f"1 of {L} layers x 1 of {B} sequences ({workload}): verify {ref.Hq}x{gamma + 1} attend_collect "
                      f"over {ref.ctx} keys {ph[0]:.2f}s + collect2 select {ph[1]:.2f}s + {gamma} draft steps "
                      f"{ph[2]:.2f}s on {threads} threads; extrapolated x{L * B}")}
    if ref.kind == "reference":
        s1, ph1 = ref.layer(threads=1)
        out["single_thread"] = {"value": round(B * (2 * gamma + 1) / (s1 * L * B), 5), "unit": "tokens/s", "cores": 1,
                                "sample": f"the same layer on 1 thread ({s1:.2f}s: verify {ph1[0]:.2f}s), "
                                          f"extrapolated x{L * B}; the reference runs single-threaded"}
    return out


def run_reference(args, rank, world, workload):
    """--impl reference: the reference's own CPU implementation (oracle/_ref) on all host threads, W
    untimed then K timed steps.  config2 (B=1): every step is the FULL iteration (all layers, no
    extrapolation).  Larger workloads: every step is one sequence x `ref_layers` layers, and `value`
    extrapolates that sample to the workload (stated in `extrapolation`)."""
    if rank != 0:
        return None
    threads = os.cpu_count() or 1
    ref = CpuReferenceSample(workload, threads)
    L, Hq, Hkv, ctx, gamma, B, desc = WORKLOADS[workload]
    full = B == 1
    n_layers = L if full else min(L, 4)
    for _ in range(args.warmup):  # warm-up steps of one layer (threads and caches warm; the run stays short)
        ref.step(1)
    secs, ph = 0.0, [0.0, 0.0, 0.0]
    for _ in range(args.steps):
        s1, p1 = ref.step(n_layers)
        secs += s1
        ph = [a + b for a, b in zip(ph, p1)]
    factor = (L * B) / n_layers
    ms_step = 1e3 * secs / args.steps  # measured wall time of one step (the sample)
    v = B * (2 * gamma + 1) / (secs / args.steps * factor)
    k = selection_k(RATIO, ctx, K_MIN)
    cores = threads if ref.kind == "reference" else 1
    sample = (f"each step: {n_layers} of {L} layers x 1 of {B} sequences ({workload}) on {threads} threads: verify "
              f"{Hq}x{gamma + 1} attend_collect over {ctx} keys + collect2 select + {gamma} draft steps per layer "
              f"(mean per step: verify {ph[0] / args.steps:.2f}s, select {ph[1] / args.steps:.2f}s, drafts "
              f"{ph[2] / args.steps:.2f}s)")
    res = {
        "metric": METRIC, "value": round(v, 4), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 2), "higher_is_better": True,
        "scaling": "weak" if workload == "config2" else "strong", "vs_baseline": None,
        "dtype": "f32/f64 (reference CPU arithmetic)", "data": "synthetic", "impl": "reference",
        "config": {"workload": f"{workload}: {desc}", "global_batch": B, "seq_len": ctx, "gamma": gamma, "k": k,
                   "selection": f"{args.strategy}, per-layer", "layers": L, "accepted": gamma},
        "cpu_baseline": {"value": round(v, 4), "unit": "tokens/s", "cores": cores, "kind": ref.kind,
                         "cpu": cpu_model(), "sample": sample},
        "e2e": {"value": round(v, 4), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not full:
        res["extrapolation"] = f"x{factor:g}: value = B*(2*gamma+1) / (ms_per_step * {factor:g})"
    return res


# dev only (SA_BENCH_SHARED_GPU=1): run N ranks on one visible GPU with a gloo process group, to check
# the multi-rank plumbing (shard plan, per-rank runs, max over ranks, rank-0 line) where only one GPU
# exists; its timings mean nothing (the ranks share the GPU), and no NCCL score exchange can run
_SHARED_GPU = os.environ.get("SA_BENCH_SHARED_GPU") == "1"


def _local_device(local_rank):
    if _SHARED_GPU:
        import torch
        return local_rank % max(1, torch.cuda.device_count())
    return local_rank


def _free_port():
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="default: config2 on 1 GPU; config3 (batch x KV-head shards, strong scaling) on N > 1")
    ap.add_argument("--shard", default=None, choices=["replica", "plan", "heads"],
                    help="replica: a full workload copy per GPU; plan: batch first, then KV heads (shard.plan); "
                         "heads: KV heads over all GPUs (shard.plan_heads). Default: replica for config1/2, plan else")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--data", default="gaussian", choices=["gaussian", "structured"],
                    help="structured: planted heavy hitters (SURVEY §8d), reports heavy_hitter_recall")
    ap.add_argument("--gamma", type=int, default=0, help="override the workload's gamma (config 5 sweep)")
    ap.add_argument("--k", type=int, default=0, help="fixed selection budget k instead of selection_k(0.07, p, 16)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the §8f next-row measurements")
    ap.add_argument("--no-headsplit", action="store_true",
                    help="N > 1: skip the config-4 KV-head split with the NCCL score exchange")
    ap.add_argument("--plan-only", action="store_true", help="print every rank's shard plan and exit (no GPU)")
    ap.add_argument("--per-kv-head", action="store_true",
                    help="per-KV-head selection (one top-k per KV head; the reference default is per layer)")
    ap.add_argument("--emulate-world", type=int, default=0,
                    help="one GPU: run rank 0's shard of an N-GPU job (per-rank work; a one-rank communicator)")
    ap.add_argument("--strategy", default="collect2", choices=sorted(STRATEGIES),
                    help="selection strategy of the iteration (the headline is collect2; the others are the "
                         "paper's variants / baselines for the overhead comparison)")
    ap.add_argument("--dev", action="append", default=[], metavar="KNOB=VALUE",
                    help="dev-only runner knob (sa_dev_set_knob), repeatable; the defaults are the product")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    # --gpus N > 1 outside torchrun: start the N ranks ourselves (one process per GPU)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    workload = args.workload or ("config2" if world == 1 else "config3")
    mode = args.shard or ("replica" if workload in ("config1", "config2") else "plan")

    if args.plan_only:  # CPU check of the launch + sharding plumbing (gloo): each rank reports its shard
        import torch.distributed as dist
        dist.init_process_group("gloo")
        sh = shard_for(workload, mode, world, rank)[0]
        obj = [None] * world
        dist.all_gather_object(obj, {"rank": rank, "world": world, "seqs": list(sh.seqs) if sh else None,
                                     "heads": [sh.heads.start, sh.heads.stop] if sh else None,
                                     "head_group": sh.head_group if sh else 1})
        if rank == 0:
            print(json.dumps({"plan": obj, "workload": workload, "shard": mode}), flush=True)
        dist.destroy_process_group()
        return

    if args.impl == "reference":
        res = run_reference(args, rank, world, workload)
        if res is not None:
            print(json.dumps(res), flush=True)
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        if _SHARED_GPU:  # dev plumbing check: every rank on the one visible GPU, host-side gloo
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    res = run_ours(args, rank, world, local_rank, workload, mode, data=args.data)
    if world > 1 and not args.no_headsplit:
        # §8e: the config-4 shape with its KV heads split over all N GPUs, so every layer's per-layer
        # selection exchanges the int64 column sums over NCCL inside the iteration graph
        try:
            hs = run_ours(args, rank, world, local_rank, "config4", "heads", steps=min(args.steps, 10),
                          warmup=3, e2e=False,
                          label=f"config4 shape, KV heads split over {world} GPUs (NCCL per-layer score exchange)")
            res["headsplit"] = {key: hs[key] for key in ("value", "unit", "ms_per_step", "config", "hbm", "comm",
                                                         "phases", "scaling") if key in hs}
        except Exception as e:  # reported, never fatal to the headline line
            res["headsplit"] = {"error": str(e)[:300]}
    if rank == 0:
        if not args.no_cpu_baseline:
            try:
                res["cpu_baseline"] = cpu_baseline(workload)
            except Exception as e:  # reported, never fatal
                res["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
        if world == 1 and not args.no_extras:
            import torch
            res["next_rows"] = next_rows(torch.device("cuda", local_rank), 1, WORKLOADS[workload][4], peaks()[0])
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
